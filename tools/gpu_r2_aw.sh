# smem carveout experiment + c0 chunk 256 with the overlapped pipeline
mkdir -p gpurun_out
for CV in -1 100; do for C in 0 1; do
  ST=50; [ $C = 0 ] && ST=1000
  PK_CARVEOUT=$CV timeout 300 python bench.py --config $C --steps $ST --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));s=d['stage_ms_per_step'];print('c$C carve $CV', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in s.items()})"
done; done
for CR in 256 512; do
  PK_CHUNK_ROWS=$CR timeout 300 python bench.py --config 0 --steps 1000 --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));s=d['stage_ms_per_step'];print('c0 chunk $CR', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in s.items()})"
done
