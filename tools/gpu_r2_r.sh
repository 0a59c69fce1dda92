mkdir -p gpurun_out
timeout 600 python tools/prof_insert_bare.py > gpurun_out/prof_ins.txt 2>&1; echo rc=$?
