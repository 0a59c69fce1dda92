mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tier.py tests/test_gpu_agents.py -q -x > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
PK_DEBUG_ASSIGN=1 timeout 600 python tools/insert_breakdown.py > gpurun_out/ins_sim.txt 2>&1; grep "pk_assign host" gpurun_out/ins_sim.txt | tail -1; tail -1 gpurun_out/ins_sim.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rerank_merge -s 4 -c 1 -o gpurun_out/rr_c1 -f python bench.py --config 1 --steps 3 --warmup 2 --no-e2e --cpu-sample 4 > gpurun_out/rr_c1.log 2>&1; echo "ncu rr rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:graph_search -s 20 -c 1 -o gpurun_out/graph_agent -f python tools/bench_agents.py --agents 4 --rows 50000 --d 1024 --rounds 2 --alpha 0.7 --ref-rounds 0 > gpurun_out/graph_agent.log 2>&1; echo "ncu graph rc=$?"
ls -la gpurun_out/*.ncu-rep
