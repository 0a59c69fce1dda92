# host arena segments registered ahead on a helper thread: tier parity, then the stream
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tier.py tests/test_gpu_executor.py tests/test_gpu_reference_suite.py tests/test_gpu_persist.py tests/test_gpu_config_scale.py -q -x -rxXf > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t.log
bash tools/gpu_r2_stream.sh
