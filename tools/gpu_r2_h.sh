# round 2: lean co-resident re-rank A/B (cfg1, cfg0), parity tests, agent profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py -q -x > gpurun_out/parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/parity.log
for L in 1 0 1; do
  PK_RERANK_LEAN=$L timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_lean$L.json 2>gpurun_out/c1_lean$L.err
  python -c "import json;d=json.load(open('gpurun_out/c1_lean$L.json'));print('c1 lean $L', round(d['value']), d['ms_per_step'], d['parity_vs_oracle'])"
  PK_RERANK_LEAN=$L timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_lean$L.json 2>gpurun_out/c0_lean$L.err
  python -c "import json;d=json.load(open('gpurun_out/c0_lean$L.json'));print('c0 lean $L', round(d['value']), d['ms_per_step'], d['parity_vs_oracle'])"
done
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 4 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_prof.json 2> gpurun_out/agents_prof.err; echo "prof rc=$?"
