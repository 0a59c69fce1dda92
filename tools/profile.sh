#!/usr/bin/env bash
# ncu evidence for the search hot path (run under gpurun, one GPU).
#   1. launch list: every kernel of a few search steps with device time
#   2. one --set full capture of the fused scan kernel (+ the coarse GEMV)
set -euo pipefail
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
ARGS="--steps 4 --warmup 2 --no-e2e --cpu-sample 4"
NCU=${NCU:-ncu}
$NCU --metrics gpu__time_duration.sum --clock-control none \
     -k regex:'scan_|dist_dense|coarse_|route_|merge_|qnorm|qprep|qswizzle|rerank|gather_rows|append_rows|stage_norms|lists_dist|shard_merge|reblock' \
     --csv --log-file "$OUT/launches.csv" python bench.py $ARGS > "$OUT/launches_bench.log" 2>&1
$NCU --set full --clock-control none --import-source on -k regex:scan_ -s 2 -c 1 \
     -o "$OUT/scan_full" -f python bench.py $ARGS > "$OUT/scan_full.log" 2>&1
$NCU --set full --clock-control none --import-source on -k regex:coarse_tc -s 2 -c 1 \
     -o "$OUT/coarse_full" -f python bench.py $ARGS > "$OUT/coarse_full.log" 2>&1
echo done
