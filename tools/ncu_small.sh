# ncu --set full captures of the small per-step kernels (pick, rerank merge, route)
mkdir -p gpurun_out
ARGS="--steps 3 --warmup 2 --no-e2e --cpu-sample 4"
for k in coarse_pick rerank_merge coarse_tc route_emit; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
     -o gpurun_out/${k}_full -f python bench.py $ARGS > gpurun_out/${k}_full.log 2>&1
  echo "$k rc=$?"
done
