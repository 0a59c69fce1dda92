mkdir -p gpurun_out
for E in 32:0.5 32:0.4 32:0.3 24:0.4 40:0.4 40:0.5 32:0.2 16:0.3; do
  PK_SCAN_EARLY=$E timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c1_e.json'));print('c1 early $E', round(d['value']), round(d['ms_per_step'],4))"
done
for K in 80 72; do
for E in 32:0.7 32:0.5 32:0.4; do
  PK_PICK_SMEM_KB=$K PK_SCAN_EARLY=$E timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c1_e.json'));print('c1 pick $K early $E', round(d['value']), round(d['ms_per_step'],4), d['stage_ms_per_step']['coarse_select'])"
done
done
PK_SCAN_EARLY=32:0.4 PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --steps 60 --no-e2e --cpu-sample 4 > /dev/null 2> gpurun_out/c1_tl.err; grep -A12 timeline gpurun_out/c1_tl.err | head -12
