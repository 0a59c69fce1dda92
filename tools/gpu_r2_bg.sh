# configs[0]: how many SMs the short-queue rule hands to the front half
mkdir -p gpurun_out
for E in 16 20 24 28 32 40 48; do
  PK_SCAN_EARLY=$E:0.3:4 timeout 300 python bench.py --config 0 --steps 2000 --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c0 early $E', round(d['value']), round(d['ms_per_step'],4))"
done
for K in 110 72; do
  PK_PICK_SMEM_KB=$K PK_SCAN_EARLY=16:0.3:4 timeout 300 python bench.py --config 0 --steps 2000 --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c0 pick $K early 16', round(d['value']), round(d['ms_per_step'],4))"
done
