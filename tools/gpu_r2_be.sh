mkdir -p gpurun_out
PK_TIME_CALLS=1 timeout 900 python tools/bench_stream.py --inserts 80000 --ref-inserts 0 --parity 8 > gpurun_out/s.json 2> gpurun_out/s.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s.json'));print({k:d[k] for k in ('insert_vectors_per_s','insert_us_per_batch_of_8','search_qps')})"
grep "calls/batch" gpurun_out/s.err
