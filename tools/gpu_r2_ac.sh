mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "overlap or async or concurrent or device_search or cfg1" > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
for D in 1 0 1 0; do
  PK_RERANK_DEFER=$D timeout 300 python bench.py --steps 50 --cpu-sample 4 > gpurun_out/c1_d.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c1_d.json'));print('c1 defer $D', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), d['parity_vs_oracle']['id_mismatch'])"
done
for D in 1 0; do
  PK_RERANK_DEFER=$D timeout 300 python bench.py --config 0 --steps 400 --cpu-sample 4 > gpurun_out/c0_d.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c0_d.json'));print('c0 defer $D', round(d['value']), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']))"
done
