# agent-path tests (batched L1 placement of inserts), the reference suites,
# a timed agent run, then the configs[0] scan experiments
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_agents.py tests/test_gpu_reference_suite.py tests/test_gpu_persist.py tests/test_gpu_sharded_store.py -q -x -rxXf > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t.log
PK_TIME_CALLS=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_t.json 2> gpurun_out/agents_t.err; echo "agents rc=$?"
python -c "import json; d=json.load(open('gpurun_out/agents_t.json')); m=d['modes']['alpha_et=0.7']; print({k: m[k] for k in ('ms_per_op','search_ms_per_query','insert8_ms','levels','early_terminated')}); [print(k, v) for k, v in list(m.get('call_ms', {}).items())[:25]]"
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_p.json 2> gpurun_out/agents_p.err; echo "agents prof rc=$?"
bash tools/gpu_r2_c0exp.sh
