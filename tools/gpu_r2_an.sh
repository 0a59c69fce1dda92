# overlapping consecutive scans (PK_SCAN_OVERLAP=1)
mkdir -p gpurun_out
PK_SCAN_OVERLAP=1 timeout 600 python -m pytest tests -m gpu -x -q -k "async_submit or back_to_back or overlap or pipelin" > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
for O in 0 1; do for E in 32:0.5 0:1 16:0.5; do for C in 1 0; do
  ST=50; [ $C = 0 ] && ST=400
  PK_SCAN_OVERLAP=$O PK_SCAN_EARLY=$E timeout 300 python bench.py --config $C --steps $ST --no-e2e --cpu-sample 0 > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));p=d['parity_vs_oracle'];print('c$C ovl $O early $E', round(d['value']), round(d['ms_per_step'],4), 'parity', p['queries'], p['id_mismatch'], p['dist_bit_mismatch'])"
done; done; done
PK_SCAN_OVERLAP=1 PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --steps 60 --no-e2e --cpu-sample 4 > /dev/null 2> gpurun_out/c1_tl.err; grep -A8 timeline gpurun_out/c1_tl.err | head -8
