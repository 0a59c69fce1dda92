mkdir -p gpurun_out
timeout 600 python tools/prof_insert.py > gpurun_out/prof_insert.txt 2>&1; echo "prof_insert rc=$?"; head -3 gpurun_out/prof_insert.txt
ACC=simulated timeout 600 python tools/prof_insert.py > gpurun_out/prof_insert_sim.txt 2>&1; echo "prof_insert sim rc=$?"; head -3 gpurun_out/prof_insert_sim.txt
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 2400 python tools/bench_stream.py > gpurun_out/stream.json 2> gpurun_out/stream.err; echo "stream rc=$?"
cat gpurun_out/stream.json; tail -5 gpurun_out/stream.err
