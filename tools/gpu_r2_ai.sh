# small-queue early release: configs[0] / [1] / [3] at the new default vs T=0
mkdir -p gpurun_out
for E in default 32:0.5:0; do
  for C in 0 1; do
    if [ $E = default ]; then unset PK_SCAN_EARLY; else export PK_SCAN_EARLY=$E; fi
    ST=50; [ $C = 0 ] && ST=400
    timeout 300 python bench.py --config $C --steps $ST --cpu-sample 4 > gpurun_out/e.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c$C early $E', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), d['parity_vs_oracle']['id_mismatch'])"
  done
done
unset PK_SCAN_EARLY
PK_RERANK_LEAN=0 timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c0 lean0', round(d['value']), round(d['ms_per_step'],4))"
timeout 900 python bench.py --config 3 --steps 10 --no-e2e --cpu-sample 4 > gpurun_out/e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c3', round(d['value']), round(d['ms_per_step'],4))"
