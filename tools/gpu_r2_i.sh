# round 2: agent path (staged kernels, count stop rule), lean re-rank with exact smem accounting
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_agents.py tests/test_gpu_graph.py tests/test_gpu_reference_suite.py tests/test_gpu_tier.py tests/test_gpu_parity.py -q -x -rxXf > gpurun_out/agent_tests.log 2>&1; rc=$?; echo "tests rc=$rc"
tail -4 gpurun_out/agent_tests.log
for L in 1 0; do
  PK_DEBUG_RERANK=1 PK_RERANK_LEAN=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --cpu-sample 4 2>&1 >/dev/null | grep "lean re-rank" | head -2
  PK_RERANK_LEAN=$L timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_lean$L.json 2>gpurun_out/c1_lean$L.err
  python -c "import json;d=json.load(open('gpurun_out/c1_lean$L.json'));print('c1 lean $L', round(d['value']), d['ms_per_step'], d['parity_vs_oracle'])"
  PK_RERANK_LEAN=$L timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_lean$L.json 2>gpurun_out/c0_lean$L.err
  python -c "import json;d=json.load(open('gpurun_out/c0_lean$L.json'));print('c0 lean $L', round(d['value']), d['ms_per_step'], d['parity_vs_oracle'])"
done
if [ $rc = 0 ]; then
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 4 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_prof.json 2> gpurun_out/agents_prof.err; echo "prof rc=$?"
python -c "import json;d=json.load(open('gpurun_out/agents_prof.json'));print(d['modes'])"
fi
