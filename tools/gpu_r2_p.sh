mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tier.py tests/test_gpu_executor.py tests/test_gpu_parity.py tests/test_gpu_sharded_insert.py tests/test_gpu_reference_suite.py -q -x > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
timeout 600 python tools/insert_breakdown.py > gpurun_out/ins_sim.txt 2>&1; tail -1 gpurun_out/ins_sim.txt
ACC=native timeout 600 python tools/insert_breakdown.py > gpurun_out/ins_nat.txt 2>&1; tail -1 gpurun_out/ins_nat.txt
