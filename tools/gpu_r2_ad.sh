mkdir -p gpurun_out
for D in 1 0; do
PK_RERANK_DEFER=$D PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --steps 60 --no-e2e --cpu-sample 4 > gpurun_out/c1_tl.json 2> gpurun_out/c1_tl$D.err
echo "defer $D"; grep -A40 "timeline" gpurun_out/c1_tl$D.err | head -22
done
PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --config 0 --steps 100 --no-e2e --cpu-sample 4 > gpurun_out/c0_tl.json 2> gpurun_out/c0_tl.err
echo "c0"; grep -A40 "timeline" gpurun_out/c0_tl.err | head -22
