mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/pytest_gpu.log
grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head -5
