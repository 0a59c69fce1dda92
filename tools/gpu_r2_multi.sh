# N>1 code path on the final tree (both ranks on the one GPU: a code-path check, never a number):
# self-launch (--gpus 2 without torchrun) and the driver's torchrun form, plus the reference arm at N=2
mkdir -p gpurun_out
PK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --config 3 > gpurun_out/multi_self.json 2> gpurun_out/multi_self.err; echo "self rc=$?"; tail -c 700 gpurun_out/multi_self.json; echo
PK_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 --impl reference > gpurun_out/multi_ref.json 2> gpurun_out/multi_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/multi_ref.json; echo
