# agent search batches: the batched list pass (pk_agent_lists) -- parity first, then timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_agents.py tests/test_gpu_graph.py tests/test_gpu_reference_suite.py tests/test_gpu_sharded_store.py -q -x -rxXf > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/t.log
PK_TIME_CALLS=1 timeout 900 python tools/bench_agents.py --rounds 4 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_e.json 2> gpurun_out/agents_e.err; echo "agents rc=$?"
python -c "import json; d=json.load(open('gpurun_out/agents_e.json')); m=d['modes']['alpha_et=0.7']; print({k: m[k] for k in ('ms_per_op','search_ms_per_query','insert8_ms')}); [print(k, v) for k, v in list(m.get('call_ms', {}).items())[:14]]"
tail -3 gpurun_out/agents_e.err
