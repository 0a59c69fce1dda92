# round 2: the new GPU test modules first (fast feedback), then the whole -m gpu suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded_store.py tests/test_gpu_agents.py tests/test_gpu_reference_suite.py tests/test_gpu_config_scale.py -q -rxXf -x ${PYTEST_ARGS:-} > gpurun_out/new_tests.log 2>&1; echo "new rc=$?"
tail -30 gpurun_out/new_tests.log
if [ -n "${FULL:-}" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"
tail -5 gpurun_out/pytest_gpu.log
fi
