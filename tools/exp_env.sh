# bench under several env settings on one box: EXP_ENVS="A=1,B=0 A=0" (comma-separated per run)
for round in 1 2; do
  for e in ${EXP_ENVS}; do
    env $(echo "$e" | tr ',' ' ') timeout 300 python bench.py --steps 300 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print('$e', round(j['value']), round(j['ms_per_step']*1e3,1), round(j['roofline']['kernel_ms_per_launch']*1e3,1), round(j['e2e']['value']), j['parity_vs_oracle']['id_mismatch'])"
  done
done
