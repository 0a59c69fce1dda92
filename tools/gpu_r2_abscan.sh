# A/B of two library builds on one box (gpurun_ab/lib_<v>.so): configs[1] and configs[0]
mkdir -p gpurun_out
for round in 1 2; do
  for v in old new; do
    cp gpurun_ab/lib_$v.so paper_2602_21477_b200/libpancake_b200.so
    for C in 1 0; do
      S=300; [ $C = 0 ] && S=2000
      timeout 300 python bench.py --config $C --steps $S --no-e2e --cpu-sample 4 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print('$v c$C', round(j['value']), round(j['ms_per_step']*1e3,1), 'scan', round(j['roofline']['kernel_ms_per_launch']*1e3,1), 'mism', j['parity_vs_oracle']['id_mismatch'], j['parity_vs_oracle']['dist_bit_mismatch'])"
    done
  done
done
cp gpurun_ab/lib_new.so paper_2602_21477_b200/libpancake_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py -q -x > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
