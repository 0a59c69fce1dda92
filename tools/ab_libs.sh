# A/B of library builds on one box: gpurun_ab/lib_<name>.so swapped in turn
for round in $(seq ${AB_ROUNDS:-2}); do
  for v in ${AB_LIBS:-head R2 R4}; do
    cp gpurun_ab/lib_$v.so paper_2602_21477_b200/libpancake_b200.so
    timeout 300 python bench.py --steps 300 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print('$v', round(j['value']), round(j['ms_per_step']*1e3,1), round(j['roofline']['kernel_ms_per_launch']*1e3,1), round(j['e2e']['value']), j['parity_vs_oracle']['id_mismatch'], {k: round(v*1e3,1) for k,v in j['stage_ms_per_step'].items()})"
  done
done
