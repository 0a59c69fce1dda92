# GPU tests, pick phase breakdown and a bench line (one gpurun call)
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
PK_DEBUG_PICK=1 timeout 300 python bench.py --steps 3 --warmup 3 2>&1 >/dev/null | grep "pick phases" | tail -2
timeout 300 python bench.py --steps 200 2>/dev/null | python -c "import json,sys; j=json.load(sys.stdin); print(round(j['value']), j['ms_per_step'], j['roofline']['kernel_ms_per_launch'], round(j['e2e']['value']), j['parity_vs_oracle'], {k: round(v*1e3,1) for k,v in j['stage_ms_per_step'].items()})"
