mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_persist.py -q > gpurun_out/tp.log 2>&1; echo "persist rc=$?"; grep -E "^E  |passed|failed" gpurun_out/tp.log | head -30
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_persist.py > gpurun_out/t.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/t.log
