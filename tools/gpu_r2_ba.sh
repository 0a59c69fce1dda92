mkdir -p gpurun_out
PK_DEBUG_ASSIGN=1 timeout 600 python tools/insert_parts.py 2>&1 | tail -16
