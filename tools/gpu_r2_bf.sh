mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "assign or insert or tier or stream" > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
PK_DEBUG_ASSIGN=1 PK_TIME_CALLS=1 timeout 900 python tools/bench_stream.py --inserts 80000 --ref-inserts 0 --parity 8 > gpurun_out/s.json 2> gpurun_out/s.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s.json'));print({k:d[k] for k in ('insert_vectors_per_s','insert_us_per_batch_of_8','search_qps','parity_vs_oracle')})"
grep "calls/batch\|pk_assign host" gpurun_out/s.err | tail -12
