# host profiles: the agent stream (cProfile) and the insert path's kernels
mkdir -p gpurun_out
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 3 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_p.json 2> gpurun_out/agents_p.err; echo "rc=$?"
ACC=native timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/ins_launches.csv python tools/insert_breakdown.py > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'P'
import csv,collections
rows=[r for r in csv.reader(open('gpurun_out/ins_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[1:]:
    try: agg[r[ki][:60]].append(float(r[vi].replace(',','')))
    except: pass
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1])): print(f"{k:60s} n={len(v)} mean={sum(v)/len(v):.0f}")
P
