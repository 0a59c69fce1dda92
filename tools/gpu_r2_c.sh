mkdir -p gpurun_out
timeout 600 python tools/insert_breakdown.py > gpurun_out/insert_breakdown.txt 2>&1; echo "breakdown rc=$?"; tail -3 gpurun_out/insert_breakdown.txt
timeout 1200 python -m pytest tests/test_gpu_graph.py tests/test_gpu_agents.py tests/test_gpu_reference_suite.py -q -rxXf -x > gpurun_out/graph_tests.log 2>&1; echo "graph rc=$?"
tail -30 gpurun_out/graph_tests.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"
tail -8 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
