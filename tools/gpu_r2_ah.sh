# configs[0]: SMs kept free of the scan for the next front half
mkdir -p gpurun_out
for E in 32:0.5 32:0.0 24:0.0 40:0.0 48:0.0 32:0.2 64:0.2 64:0.0; do
  PK_SCAN_EARLY=$E timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c0_e.json'));print('c0 early $E', round(d['value']), round(d['ms_per_step'],4), d['parity_vs_oracle']['id_mismatch'])"
done
for S in 116 124; do
  PK_SCAN_SMS=$S PK_SCAN_EARLY=0:1 timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c0_e.json'));print('c0 sms $S', round(d['value']), round(d['ms_per_step'],4))"
done
PK_SCAN_EARLY=32:0.0 PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --config 0 --steps 60 --no-e2e --cpu-sample 4 > /dev/null 2> gpurun_out/c0_tl.err; grep -A12 timeline gpurun_out/c0_tl.err | head -8
