# configs[1]: SMs reserved for the front half / re-rank (scan grid below 148)
mkdir -p gpurun_out
for S in 148 140 132 124 116; do
  for E in 0:1 32:0.5; do
    PK_SCAN_SMS=$S PK_SCAN_EARLY=$E timeout 300 python bench.py --config 1 --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/e.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c1 sms $S early $E', round(d['value']), round(d['ms_per_step'],4), 'scan', round(d['stage_ms_per_step']['scan'],4))"
  done
done
