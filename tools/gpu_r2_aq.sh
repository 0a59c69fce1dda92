mkdir -p gpurun_out
for C in 0 1; do
  ST=2000; [ $C = 1 ] && ST=200
  PK_BENCH_HOST_TIMES=1 PK_DEBUG_SUBMIT=1 timeout 300 python bench.py --config $C --steps $ST --cpu-sample 0 --no-parity > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c$C', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']))"
  grep "host us" gpurun_out/e.err | tail -3
done
