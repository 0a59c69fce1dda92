# every BASELINE config's measurement on one B200 (run under gpurun); outputs in gpurun_out/cfg_*.json
mkdir -p gpurun_out
timeout 600 python bench.py --rows 100000 --d 384 --nlist 256 --nprobe 16 --batch 32 --steps 300 > gpurun_out/cfg1.json 2> gpurun_out/cfg1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --impl reference --rows 100000 --d 384 --nlist 256 --nprobe 16 --batch 32 --steps 3 --warmup 3 > gpurun_out/cfg1_ref.json 2> gpurun_out/cfg1_ref.err; echo "cfg1 ref rc=$?"
timeout 1200 python bench.py --rows 10000000 --nlist 8192 --steps 20 --warmup 3 > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"
timeout 1200 python tools/bench_agents.py > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; echo "cfg3 rc=$?"
timeout 1200 python tools/bench_stream.py --inserts 20000 --search-every 64 > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err; echo "cfg5 rc=$?"
