mkdir -p gpurun_out
PK_DEBUG_ASSIGN=1 timeout 600 python tools/insert_parts.py 2>&1 | tail -12
timeout 1500 python -m pytest tests -m gpu -q -x -k "tier or insert or store or agents or persist or reference_suite or parity" > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
