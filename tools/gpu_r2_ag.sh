# full GPU suite on the current tree, c0 timeline, insert profiles (native tier)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t.log
PK_DEBUG_TIMELINE=1 timeout 300 python bench.py --config 0 --steps 60 --no-e2e --cpu-sample 4 > /dev/null 2> gpurun_out/c0_tl.err; grep -A12 timeline gpurun_out/c0_tl.err | head -12
ACC=native PK_DEBUG_ASSIGN=1 timeout 600 python tools/insert_breakdown.py > gpurun_out/ins_nat.txt 2> gpurun_out/ins_nat.err; cat gpurun_out/ins_nat.txt; grep pk_assign gpurun_out/ins_nat.err | tail -2
ACC=native timeout 600 python tools/prof_insert_bare.py > gpurun_out/prof_ins.txt 2>&1; head -75 gpurun_out/prof_ins.txt
