# configs[2] 8 rounds, alpha 0.7: call timers + buffer / row-store growth events
mkdir -p gpurun_out
PK_DEBUG_GROW=1 PK_TIME_CALLS=1 timeout 1200 python tools/bench_agents.py --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_g.json 2> gpurun_out/agents_g.err; echo "agents rc=$?"
python -c "import json; d=json.load(open('gpurun_out/agents_g.json')); m=d['modes']['alpha_et=0.7']; print({k: m[k] for k in ('ms_per_op','search_ms_per_query','insert8_ms')}); [print(k, v) for k, v in list(m.get('call_ms', {}).items())[:12]]"
grep -c "grow" gpurun_out/agents_g.err; grep "row store grow" gpurun_out/agents_g.err | tail -8; grep "pinned buffer grow" gpurun_out/agents_g.err | tail -5
