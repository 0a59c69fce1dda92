# round 2: agent path rewrite -- agent tests, reference suite, small + full agent bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_agents.py tests/test_gpu_graph.py tests/test_gpu_reference_suite.py tests/test_gpu_tier.py -q -x -rxXf > gpurun_out/agent_tests.log 2>&1; rc=$?; echo "agent tests rc=$rc"
tail -30 gpurun_out/agent_tests.log
timeout 900 python tools/bench_agents.py --agents 4 --rows 20000 --d 256 --rounds 4 --alpha 0.7 > gpurun_out/agents_small.json 2> gpurun_out/agents_small.err; echo "small rc=$?"
tail -3 gpurun_out/agents_small.err
if [ $rc = 0 ]; then
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 1500 python tools/bench_agents.py > gpurun_out/agents_full.json 2> gpurun_out/agents_full.err; echo "agents full rc=$?"
cat gpurun_out/agents_full.json
fi
