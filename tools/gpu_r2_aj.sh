mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "async_submit or back_to_back" > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
for D in 2 3 4; do for C in 0 1; do
  ST=50; [ $C = 0 ] && ST=400
  PK_BENCH_E2E_DEPTH=$D timeout 300 python bench.py --config $C --steps $ST --cpu-sample 4 > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c$C depth $D', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']))"
done; done
