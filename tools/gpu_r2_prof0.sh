# host profile of the agent path with early termination off (alpha_et 0): every search scans its lists
mkdir -p gpurun_out
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.0 --ref-rounds 0 > gpurun_out/agents_p0.json 2> gpurun_out/agents_p0.err; echo "rc=$?"
grep -A28 "tottime" gpurun_out/agents_p0.err | head -30
grep -A30 "cumulative" gpurun_out/agents_p0.err | sed -n 1,34p
