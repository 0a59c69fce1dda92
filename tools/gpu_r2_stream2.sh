# configs[4] stream with the in-place host arena (+ huge-page advice), and THP settings of the box
mkdir -p gpurun_out
cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag 2>&1
bash tools/gpu_r2_stream.sh
