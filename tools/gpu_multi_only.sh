mkdir -p gpurun_out
PK_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --rows 300000 --nlist 256 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench2 rc=$?"
cat gpurun_out/bench2.json; grep -v "^W1\|^  warn" gpurun_out/bench2.err | tail -30
