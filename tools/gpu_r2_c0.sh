# configs[0] scan experiments: CTA end spread, chunk size, selection cost
mkdir -p gpurun_out
for CR in 512 256; do
  PK_CHUNK_ROWS=$CR PK_DEBUG_SCAN_TIMES=1 timeout 300 python bench.py --config 0 --steps 8 --warmup 3 --no-e2e --cpu-sample 4 > /dev/null 2> gpurun_out/c0_t$CR.err
  echo "chunk $CR"; grep "scan CTA" gpurun_out/c0_t$CR.err | tail -4
  PK_CHUNK_ROWS=$CR timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c0_e.json'));print('c0 chunk $CR', round(d['value']), round(d['ms_per_step'],4), d['stage_ms_per_step'], d['parity_vs_oracle'])"
done
PK_DEBUG_SCAN_NOSELECT=1 timeout 300 python bench.py --config 0 --steps 400 --no-e2e --no-parity --cpu-sample 4 > gpurun_out/c0_e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/c0_e.json'));print('c0 noselect', round(d['value']), round(d['ms_per_step'],4), d['stage_ms_per_step'])"
PK_DEBUG_SCAN_NOSELECT=1 PK_DEBUG_SCAN_TIMES=1 timeout 300 python bench.py --config 0 --steps 8 --warmup 3 --no-e2e --no-parity --cpu-sample 4 > /dev/null 2> gpurun_out/c0_tn.err
grep "scan CTA" gpurun_out/c0_tn.err | tail -3
for E in 32:0.5 0:1; do
PK_SCAN_EARLY=$E timeout 300 python bench.py --config 1 --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/c1_e.json'));print('c1 early $E', round(d['value']), round(d['ms_per_step'],4))"
done
