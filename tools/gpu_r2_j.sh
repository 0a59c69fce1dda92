# round 2: lean re-rank grid sweep, agent_read phase times at configs[2] scale
mkdir -p gpurun_out
for C in "0 x" "1 148" "1 64" "1 32" "1 16"; do
  set -- $C
  PK_RERANK_LEAN=$1 PK_RERANK_LEAN_CTAS=$2 timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c1_sw.json'));print('c1 lean $1 ctas $2', round(d['value']), round(d['ms_per_step'],4))"
  PK_RERANK_LEAN=$1 PK_RERANK_LEAN_CTAS=$2 timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_sw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c0_sw.json'));print('c0 lean $1 ctas $2', round(d['value']), round(d['ms_per_step'],4))"
done
PK_DEBUG_AGENT=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_dbg.json 2> gpurun_out/agents_dbg.err; echo "agents dbg rc=$?"
grep "agent_read device" gpurun_out/agents_dbg.err | tail -3
python -c "import json;d=json.load(open('gpurun_out/agents_dbg.json'));print(d['modes'])"
