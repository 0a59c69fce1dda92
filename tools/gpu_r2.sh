# round-2 GPU check: gpu tests, bench configs[1] + configs[3] (1 GPU), the
# 2-rank strong-scaling code path on one GPU, host facts
mkdir -p gpurun_out
free -g > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; nvidia-smi -L >> gpurun_out/host.txt
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench c1 rc=$?"
cat gpurun_out/bench_c1.json; tail -3 gpurun_out/bench_c1.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_c1_ref.json 2> gpurun_out/bench_c1_ref.err; echo "ref c1 rc=$?"
cat gpurun_out/bench_c1_ref.json; tail -3 gpurun_out/bench_c1_ref.err
if [ -z "${SKIP_C3:-}" ]; then
timeout 900 python bench.py --config 3 --steps 20 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?"
cat gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
PK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config 3 --rows 2000000 --nlist 2048 --steps 10 > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err; echo "share2 rc=$?"
cat gpurun_out/bench_share2.json; tail -5 gpurun_out/bench_share2.err
fi
