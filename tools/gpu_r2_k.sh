# round 2: warp graph walk; agent tests; cfg1/cfg0 defaults; agent bench profile + phases
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_agents.py tests/test_gpu_reference_suite.py tests/test_gpu_parity.py tests/test_gpu_sharded_store.py -q -x -rxXf > gpurun_out/agent_tests.log 2>&1; rc=$?; echo "tests rc=$rc"
tail -4 gpurun_out/agent_tests.log
timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/c1.json'));print('c1', round(d['value']), round(d['ms_per_step'],4), d['parity_vs_oracle'])"
timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/c0.json'));print('c0', round(d['value']), round(d['ms_per_step'],4), d['parity_vs_oracle'])"
if [ $rc = 0 ]; then
PK_DEBUG_AGENT=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_dbg.json 2> gpurun_out/agents_dbg.err; echo "agents dbg rc=$?"
grep "agent_read device" gpurun_out/agents_dbg.err | tail -1
python -c "import json;d=json.load(open('gpurun_out/agents_dbg.json'));print(d['modes'])"
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_prof.json 2> gpurun_out/agents_prof.err; echo "prof rc=$?"
fi
