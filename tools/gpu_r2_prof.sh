# round 2: reference suites against the drop-in + ncu evidence per workload
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_reference_suite.py -q -rxXs > gpurun_out/refsuite.log 2>&1; echo "refsuite rc=$?"
tail -25 gpurun_out/refsuite.log
K='scan_|dist_dense|coarse_|route_|merge_|qnorm|qprep|rerank|shard_merge'
for C in 1 0; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv \
     --log-file gpurun_out/launches_c$C.csv python bench.py --config $C --steps 4 --warmup 2 --no-e2e --cpu-sample 4 > gpurun_out/launches_c$C.log 2>&1
  echo "launches c$C rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_tc -s 2 -c 1 \
     -o gpurun_out/scan_c$C -f python bench.py --config $C --steps 3 --warmup 2 --no-e2e --cpu-sample 4 > gpurun_out/scan_c$C.log 2>&1
  echo "scan c$C rc=$?"
done
for KN in coarse_pick rerank_merge coarse_tc; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KN -s 2 -c 1 \
     -o gpurun_out/${KN}_c1 -f python bench.py --config 1 --steps 3 --warmup 2 --no-e2e --cpu-sample 4 > gpurun_out/${KN}_c1.log 2>&1
  echo "$KN rc=$?"
done
timeout 900 ncu --set full --clock-control none -k regex:scan_tc -s 2 -c 1 \
   -o gpurun_out/scan_c3 -f python bench.py --config 3 --steps 3 --warmup 2 --no-e2e --no-parity > gpurun_out/scan_c3.log 2>&1
echo "scan c3 rc=$?"
cuobjdump -sass -fun coarse_pick_kernel paper_2602_21477_b200/libpancake_b200.so > gpurun_out/sass_pick.txt 2>&1 || true
ls -la gpurun_out/*.ncu-rep
