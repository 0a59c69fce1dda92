# configs[0] scan experiments: where does the 32-query step go (timing only; the
# PK_DEBUG_SCAN_* runs produce wrong results by design)
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config 0 --steps 400 --no-e2e --cpu-sample 4 > gpurun_out/c0x_$tag.json 2> gpurun_out/c0x_$tag.err; echo "$tag rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/c0x_$tag.json').read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'scan', round(d['roofline']['kernel_ms_per_launch']*1e3,1))" 2>&1)"; }
run base X=1
run noselect PK_DEBUG_SCAN_NOSELECT=1
run early0 PK_SCAN_EARLY=0:1
run early0ns PK_SCAN_EARLY=0:1 PK_DEBUG_SCAN_NOSELECT=1
run times PK_DEBUG_SCAN_TIMES=1
grep "scan CTA times" gpurun_out/c0x_times.err | tail -5
run times1 PK_DEBUG_SCAN_TIMES=1 PK_DEBUG_SCAN_NOSELECT=1
grep "scan CTA times" gpurun_out/c0x_times1.err | tail -3
run times2 PK_DEBUG_SCAN_TIMES=1 PK_SCAN_EARLY=0:1
grep "scan CTA times" gpurun_out/c0x_times2.err | tail -3
