# Round 2 measurement pass: every BASELINE config through its tool, ncu
# evidence per workload; outputs in gpurun_out/ (copied to profiles/ by hand,
# tools/ncu_summary.py for the ncu summaries).
#   V=v2 bash tools/gpu_r2_final.sh
set -u
V=${V:-v5}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
# configs[1] (the headline), its reference arm, configs[0], configs[3] on one GPU
timeout 600 python bench.py --steps 50 > gpurun_out/r02_${V}_c1_bench.json 2> gpurun_out/c1.err; echo "c1 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02_${V}_c1_bench_ref.json 2> gpurun_out/c1r.err; echo "c1 ref rc=$?"
timeout 600 python bench.py --config 0 --steps 2000 > gpurun_out/r02_${V}_c0_bench.json 2> gpurun_out/c0.err; echo "c0 rc=$?"
timeout 600 python bench.py --config 0 --impl reference --steps 5 --warmup 3 > gpurun_out/r02_${V}_c0_bench_ref.json 2> gpurun_out/c0r.err; echo "c0 ref rc=$?"
timeout 900 python bench.py --config 3 --steps 20 > gpurun_out/r02_${V}_c3_1gpu_bench.json 2> gpurun_out/c3.err; echo "c3 rc=$?"
# configs[2]: agents, with the reference Store on the same stream
timeout 1800 python tools/bench_agents.py > gpurun_out/r02_${V}_c2_agents.json 2> gpurun_out/c2.err; echo "c2 rc=$?"
# configs[4]: 500K-insert stream with the native tier, reference simulated tier beside it
timeout 2400 python tools/bench_stream.py > gpurun_out/r02_${V}_c4_stream.json 2> gpurun_out/c4.err; echo "c4 rc=$?"
# ncu: launch lists + full captures (scan per workload, the exact chains, the agent kernels)
K='scan_|dist_dense|coarse_|route_|merge_|qnorm|qprep|rerank|shard_merge'
for C in 1 0; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv \
     --log-file gpurun_out/r02_${V}_launches_c$C.csv python bench.py --config $C --steps 4 --warmup 2 --no-e2e --cpu-sample 4 > /dev/null 2>&1
  echo "launches c$C rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_tc -s 2 -c 1 \
     -o gpurun_out/scan_c$C -f python bench.py --config $C --steps 3 --warmup 2 --no-e2e --cpu-sample 4 > /dev/null 2>&1
  echo "scan c$C rc=$?"
done
for KN in coarse_pick rerank_merge coarse_tc; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KN -s 2 -c 1 \
     -o gpurun_out/${KN}_c1 -f python bench.py --config 1 --steps 3 --warmup 2 --no-e2e --cpu-sample 4 > /dev/null 2>&1
  echo "$KN rc=$?"
done
for KN in graph_search probe_lists gather_dist l1_place; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KN -s 40 -c 1 \
     -o gpurun_out/${KN}_c2 -f python tools/bench_agents.py --agents 16 --rows 250000 --rounds 2 --alpha 0.7 --ref-rounds 0 > /dev/null 2>&1
  echo "$KN rc=$?"
done
ls -la gpurun_out/*.ncu-rep
