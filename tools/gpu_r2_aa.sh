mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_agents.py tests/test_gpu_reference_suite.py tests/test_gpu_sharded_store.py -q -x > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_t.json 2> gpurun_out/agents_t.err; echo "rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/agents_t.json'))
for k,v in d['modes'].items():
  print(k, {x: v[x] for x in ('ms_per_op','search_ms_per_query','insert8_ms')})
"
