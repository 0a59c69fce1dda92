# final tree: smoke, the whole -m gpu suite, configs[2] with the reference Store beside it, configs[4]
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -rxXfs > gpurun_out/pytest_gpu.log 2>&1; echo "full rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 1800 python tools/bench_agents.py > gpurun_out/r02_v6_c2_agents.json 2> gpurun_out/c2.err; echo "c2 rc=$?"
tail -4 gpurun_out/c2.err | cut -c1-400
timeout 2400 python tools/bench_stream.py > gpurun_out/r02_v6_c4_stream.json 2> gpurun_out/c4.err; echo "c4 rc=$?"
python -c "import json; s=json.load(open('gpurun_out/r02_v6_c4_stream.json')); print(s['insert_vectors_per_s'], s['insert_us_per_batch_of_8'], s['parity_vs_oracle'], s['same_answers_as_reference_at_its_sample'])"
