# round 2 re-entry check: the whole -m gpu suite, smoke, a short configs[1] bench
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/host.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py --steps 20 > gpurun_out/c1_bench.json 2> gpurun_out/c1.err; echo "c1 rc=$?"; cat gpurun_out/c1_bench.json | head -c 600; echo
timeout 1800 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"
tail -8 gpurun_out/pytest_gpu.log
