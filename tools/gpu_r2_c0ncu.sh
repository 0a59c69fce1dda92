# configs[0] scan: one ncu --set full capture with source, for per-line stall samples
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_tc -s 20 -c 1 \
   -o gpurun_out/scan_c0x -f python bench.py --config 0 --steps 30 --warmup 3 --no-e2e --cpu-sample 4 > gpurun_out/scan_c0x.log 2>&1
echo "ncu rc=$?"
