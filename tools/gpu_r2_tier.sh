# host arena grown in place (reserved range, registered segments): tier parity, then the stream
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tier.py tests/test_gpu_executor.py tests/test_gpu_reference_suite.py tests/test_gpu_persist.py -q -x -rxXf > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t.log
bash tools/gpu_r2_stream.sh
bash tools/gpu_r2_agentgrow.sh
