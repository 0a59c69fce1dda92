# alternating front streams (PK_FRONT_OVERLAP=1)
mkdir -p gpurun_out
PK_FRONT_OVERLAP=1 timeout 600 python -m pytest tests -m gpu -x -q -k "async_submit or back_to_back or overlap or pipelin" > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
for F in 0 1; do for C in 0 1; do
  ST=50; [ $C = 0 ] && ST=1000
  PK_FRONT_OVERLAP=$F timeout 300 python bench.py --config $C --steps $ST --cpu-sample 0 > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));p=d['parity_vs_oracle'];print('c$C front_ovl $F', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'parity', p['queries'], p['id_mismatch'], p['dist_bit_mismatch'])"
done; done
