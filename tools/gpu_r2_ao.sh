# overlapping scans: early-release sweep, defer on/off, c3 / e2e check
mkdir -p gpurun_out
export PK_SCAN_OVERLAP=1
for E in 32:0.5 24:0.5 48:0.5 64:0.5 32:0.3 32:0.7 48:0.3; do for C in 1 0; do
  ST=50; [ $C = 0 ] && ST=400
  PK_SCAN_EARLY=$E timeout 300 python bench.py --config $C --steps $ST --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c$C early $E', round(d['value']), round(d['ms_per_step'],4))"
done; done
for C in 1 0; do
  ST=50; [ $C = 0 ] && ST=400
  PK_RERANK_DEFER=0 timeout 300 python bench.py --config $C --steps $ST --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c$C defer0', round(d['value']), round(d['ms_per_step'],4))"
  timeout 300 python bench.py --config $C --steps $ST --cpu-sample 4 > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c$C e2e', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']))"
done
timeout 900 python bench.py --config 3 --steps 10 --no-e2e --cpu-sample 4 > gpurun_out/e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c3', round(d['value']), round(d['ms_per_step'],4), d['parity_vs_oracle'])"
