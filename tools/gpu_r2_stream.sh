# configs[4] stream: where the per-batch time goes at 500K inserts (call timers, arena growth)
mkdir -p gpurun_out
PK_DEBUG_GROW=1 PK_TIME_CALLS=1 timeout 1500 python tools/bench_stream.py --ref-inserts 0 > gpurun_out/stream_t.json 2> gpurun_out/stream_t.err; echo "stream rc=$?"
grep -E "grow|calls/batch" gpurun_out/stream_t.err | head -30
python -c "import json; d=json.load(open('gpurun_out/stream_t.json')); print(d['insert_vectors_per_s'], d['insert_us_per_batch_of_8'], d['search_qps'])"
