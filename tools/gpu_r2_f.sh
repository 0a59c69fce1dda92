# round 2: full-scale agent profile + cfg0/cfg1 phase timings and chunk experiments
mkdir -p gpurun_out
PK_PROFILE_OPS=1 timeout 900 python tools/bench_agents.py --rounds 4 --alpha 0.7 --ref-rounds 0 > gpurun_out/agents_prof.json 2> gpurun_out/agents_prof.err; echo "prof rc=$?"
for C in 0 1; do
  PK_DEBUG_RERANK=1 PK_DEBUG_PICK=1 PK_DEBUG_SCAN_TIMES=1 timeout 300 python bench.py --config $C --steps 6 --warmup 3 --no-e2e --cpu-sample 4 > gpurun_out/dbg_c$C.json 2> gpurun_out/dbg_c$C.err; echo "dbg c$C rc=$?"
  grep -E "rerank phases|pick|scan CTA" gpurun_out/dbg_c$C.err | tail -6
done
for CH in 256 1024; do
  PK_CHUNK_ROWS=$CH timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_ch$CH.json 2>/dev/null; echo "c0 chunk $CH rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/c0_ch$CH.json'));print('$CH', d['value'], d['ms_per_step'], d['stage_ms_per_step'])"
done
for E in 0:1 16:0.5 64:0.5; do
  PK_SCAN_EARLY=$E timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0_e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c0_e.json'));print('early $E', d['value'], d['ms_per_step'])"
done
