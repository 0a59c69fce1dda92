# host profile of the agent path (cProfile; relative self times only)
mkdir -p gpurun_out
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 4 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_p.json 2> gpurun_out/agents_p.err; echo "agents prof rc=$?"
grep -A40 "tottime" gpurun_out/agents_p.err | head -45
