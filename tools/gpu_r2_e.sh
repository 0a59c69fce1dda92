# round 2: agent workload (configs[2]) small profile + parity vs reference, then the full config
mkdir -p gpurun_out
free -g > gpurun_out/host_mem.txt; df -h /tmp >> gpurun_out/host_mem.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k nprobe_above > gpurun_out/fix.log 2>&1; echo "fix rc=$?"; tail -2 gpurun_out/fix.log
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --agents 4 --rows 20000 --d 256 --rounds 4 --alpha 0.7 > gpurun_out/agents_small.json 2> gpurun_out/agents_small.err; echo "small rc=$?"
cat gpurun_out/agents_small.json; grep -v "^ " gpurun_out/agents_small.err | tail -5
timeout 2400 python tools/bench_agents.py > gpurun_out/agents_full.json 2> gpurun_out/agents_full.err; echo "full rc=$?"
cat gpurun_out/agents_full.json; tail -5 gpurun_out/agents_full.err
