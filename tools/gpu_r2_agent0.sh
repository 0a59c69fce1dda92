# alpha_et 0: per-phase device time of pk_agent_read and growth events
mkdir -p gpurun_out
PK_DEBUG_AGENT=1 PK_DEBUG_GROW=1 PK_TIME_CALLS=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.0 --ref-rounds 0 > gpurun_out/agents_d0.json 2> gpurun_out/agents_d0.err; echo "rc=$?"
grep "agent_read device" gpurun_out/agents_d0.err | tail -2
grep "row store grow" gpurun_out/agents_d0.err | tail -4
python -c "import json; d=json.load(open('gpurun_out/agents_d0.json')); m=d['modes']['alpha_et=0.0']; print({k: m[k] for k in ('ms_per_op','search_ms_per_query')}); [print(k, v) for k, v in list(m.get('call_ms', {}).items())[:6]]"
