mkdir -p gpurun_out
timeout 2400 python tools/bench_stream.py > gpurun_out/r02_v2_c4_stream.json 2> gpurun_out/c4.err; echo "c4 rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02_v2_c4_stream.json'))
print({k:d[k] for k in ('insert_vectors_per_s','insert_us_per_batch_of_8','search_qps','pcie_gbs_effective','parity_vs_oracle','same_answers_as_reference_at_its_sample')})
"
for U in 0 1; do
  PK_RERANK_UQ=$U timeout 300 python bench.py --steps 50 --no-e2e --cpu-sample 4 > gpurun_out/c1_uq.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c1_uq.json'));print('c1 uq $U', round(d['value']), round(d['ms_per_step'],4), d['stage_ms_per_step']['merge_out'], d['screen_candidates_per_query']['rows_reranked_exactly'], d['parity_vs_oracle'])"
done
