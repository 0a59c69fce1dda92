# agent path: per-phase device time of pk_agent_read and per-call host timers
mkdir -p gpurun_out
PK_DEBUG_AGENT=1 PK_TIME_CALLS=1 timeout 900 python tools/bench_agents.py --rounds 4 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_d.json 2> gpurun_out/agents_d.err; echo "agents rc=$?"
grep "agent_read device" gpurun_out/agents_d.err | tail -3
python -c "import json; d=json.load(open('gpurun_out/agents_d.json')); m=d['modes']['alpha_et=0.7']; print({k: m[k] for k in ('ms_per_op','search_ms_per_query','insert8_ms')}); [print(k, v) for k, v in list(m.get('call_ms', {}).items())[:14]]"
PK_TIME_CALLS=1 timeout 900 python tools/bench_agents.py --rounds 4 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_e.json 2> gpurun_out/agents_e.err; echo "agents rc=$?"
python -c "import json; d=json.load(open('gpurun_out/agents_e.json')); m=d['modes']['alpha_et=0.7']; print({k: m[k] for k in ('ms_per_op','search_ms_per_query','insert8_ms')}); [print(k, v) for k, v in list(m.get('call_ms', {}).items())[:14]]"
