# pipelining check: the overlap-safety tests, then bench with and without the front-half overlap
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for p in 1 0; do
  PK_PIPELINE=$p timeout 300 python bench.py --steps 200 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print('pipeline', $p, round(j['value']), j['ms_per_step'], j['roofline']['kernel_ms_per_launch'], round(j['e2e']['value']), j['parity_vs_oracle'])"
done
