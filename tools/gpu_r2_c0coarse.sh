# configs[0]: coarse stage variants x reserved front SMs (A/B on one box)
mkdir -p gpurun_out
for round in 1 2; do
for V in "tc 32:0.3:4" "exact 32:0.3:4" "exact 24:0.3:4" "exact 16:0.3:4" "tf32 32:0.3:4"; do
  set -- $V
  PK_COARSE=$1 PK_SCAN_EARLY=$2 timeout 300 python bench.py --config 0 --steps 2000 --no-e2e --cpu-sample 4 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print('$1 $2', round(j['value']), round(j['ms_per_step']*1e3,1), 'scan', round(j['roofline']['kernel_ms_per_launch']*1e3,1), 'mism', j['parity_vs_oracle']['id_mismatch'], j['parity_vs_oracle']['dist_bit_mismatch'], {k: round(v*1e3,1) for k,v in j['stage_ms_per_step'].items()})"
done
done
