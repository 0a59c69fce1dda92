mkdir -p gpurun_out
for ST in 400 400 1000 2000; do
  PK_BENCH_HOST_TIMES=1 timeout 300 python bench.py --config 0 --steps $ST --cpu-sample 0 --no-parity > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c0 steps $ST', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']))"
  grep "host us" gpurun_out/e.err | tail -2
done
PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --config 0 --steps 60 --no-e2e --cpu-sample 0 > /dev/null 2> gpurun_out/c0_tl.err; grep -A10 timeline gpurun_out/c0_tl.err | head -10
