mkdir -p gpurun_out
PK_BENCH_HOST_TIMES=1 PK_DEBUG_SUBMIT=2 timeout 300 python bench.py --config 0 --steps 2000 --cpu-sample 0 --no-parity > gpurun_out/e.json 2> gpurun_out/e.err
python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c0', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']))"
grep -A1 "host us" gpurun_out/e.err | tail -4
