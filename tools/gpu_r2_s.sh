mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/insert_breakdown.py > gpurun_out/ins_sim.txt 2>&1; tail -1 gpurun_out/ins_sim.txt
ACC=native timeout 600 python tools/insert_breakdown.py > gpurun_out/ins_nat.txt 2>&1; tail -1 gpurun_out/ins_nat.txt
