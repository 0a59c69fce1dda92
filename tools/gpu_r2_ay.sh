# hardware work queues: CUDA_DEVICE_MAX_CONNECTIONS 8 (default) vs 16 / 32
mkdir -p gpurun_out
for MC in 8 16 32; do for C in 0 1; do
  ST=50; [ $C = 0 ] && ST=1000
  CUDA_DEVICE_MAX_CONNECTIONS=$MC timeout 300 python bench.py --config $C --steps $ST --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c$C conn $MC', round(d['value']), round(d['ms_per_step'],4))"
done; done
CUDA_DEVICE_MAX_CONNECTIONS=32 PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --config 0 --steps 60 --no-e2e --cpu-sample 0 --no-parity > /dev/null 2> gpurun_out/c0_tl.err; grep -A8 timeline gpurun_out/c0_tl.err | head -8
