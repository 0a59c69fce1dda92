# row store reserved per registered agent: agent parity, then configs[2] (both alpha) with growth events
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_agents.py tests/test_gpu_sharded_store.py tests/test_gpu_reference_suite.py tests/test_gpu_persist.py tests/test_abi.py -q -x -rxXf > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
PK_DEBUG_GROW=1 timeout 1500 python tools/bench_agents.py --ref-rounds 0 > gpurun_out/agents_r.json 2> gpurun_out/agents_r.err; echo "agents rc=$?"
grep -c "row store grow" gpurun_out/agents_r.err; grep "row store grow" gpurun_out/agents_r.err | sort -t: -k2 -n | tail -3
python -c "import json; d=json.load(open('gpurun_out/agents_r.json')); [print(a, {k: round(m[k],3) for k in ('ms_per_op','search_ms_per_query','insert8_ms')}) for a, m in d['modes'].items()]"
