# round 2 re-entry: full -m gpu suite, smoke, bench configs[1] + reference arm
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/host.txt; nproc >> gpurun_out/host.txt
timeout 1800 python -m pytest tests -m gpu -q -rxXf > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"
tail -25 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench c1 rc=$?"
cat gpurun_out/bench_c1.json; tail -3 gpurun_out/bench_c1.err
timeout 600 python bench.py --config 0 --steps 200 > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err; echo "bench c0 rc=$?"
cat gpurun_out/bench_c0.json; tail -3 gpurun_out/bench_c0.err
