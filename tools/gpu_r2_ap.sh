# overlapping scans as the default: full GPU suite, early-release confirmation
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t.log
for E in 32:0.3 32:0.2 32:0.4 40:0.3 48:0.4; do
  PK_SCAN_EARLY=$E timeout 300 python bench.py --config 1 --steps 50 --no-e2e --cpu-sample 0 --no-parity > gpurun_out/e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e.json'));print('c1 early $E', round(d['value']), round(d['ms_per_step'],4))"
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
