mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "async_submit or scope or store" > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
for ST in 400 2000; do
PK_BENCH_HOST_TIMES=1 PK_DEBUG_SUBMIT=1 timeout 300 python bench.py --config 0 --steps $ST --cpu-sample 0 --no-parity > gpurun_out/e.json 2> gpurun_out/e.err
python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c0', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']))"
grep "host us" gpurun_out/e.err | tail -2
done
