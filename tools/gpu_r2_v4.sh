# v4 pass of the paths changed since v3 (host policy of the agent path, insert path):
# configs[2] agents and configs[4] stream, each with the reference package beside it
set -u
V=${V:-v4}
mkdir -p gpurun_out
timeout 1800 python tools/bench_agents.py > gpurun_out/r02_${V}_c2_agents.json 2> gpurun_out/c2.err; echo "c2 rc=$?"
timeout 2400 python tools/bench_stream.py > gpurun_out/r02_${V}_c4_stream.json 2> gpurun_out/c4.err; echo "c4 rc=$?"
