mkdir -p gpurun_out
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_prof.json 2> gpurun_out/agents_prof.err; echo "prof rc=$?"
