mkdir -p gpurun_out
timeout 600 python tools/insert_parts.py 2>&1 | tail -10
ACC=native timeout 600 python tools/insert_breakdown.py 2>&1 | tail -1
timeout 900 python tools/bench_stream.py --inserts 80000 --ref-inserts 0 --parity 8 > gpurun_out/s.json 2> gpurun_out/s.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s.json'));print({k:d[k] for k in ('insert_vectors_per_s','insert_us_per_batch_of_8','search_qps','parity_vs_oracle')})"
