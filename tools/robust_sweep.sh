# robustness sweep of the cfg2 index: bigger batches, deeper probes, larger k (parity vs the oracle on a sample)
for args in "--batch 1024" "--batch 4096 --steps 20" "--nprobe 128 --steps 50" "--k 64 --steps 50" "--batch 1 --steps 300" "--nprobe 1 --k 1"; do
  timeout 600 python bench.py $args --cpu-sample 8 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print('$args', round(j['value']), round(j['ms_per_step']*1e3,1), round(j['e2e']['value']), j['parity_vs_oracle'])" || echo "$args FAILED"
done
