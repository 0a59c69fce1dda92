mkdir -p gpurun_out
for E in 32:0.7 32:0.6 32:0.5 48:0.7 48:0.6 64:0.7 64:0.6 64:0.5 96:0.7 96:0.8; do
  PK_SCAN_EARLY=$E timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c1_e.json'));print('c1 early $E', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_launch'],4))"
done
for E in 32:0.7 16:0.5 32:0.5 64:0.5 64:0.7; do
  PK_SCAN_EARLY=$E timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c0_e.json'));print('c0 early $E', round(d['value']), round(d['ms_per_step'],4))"
done
