# ncu --set full of one kernel (regex $1) during a short bench run
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 2 -c 1 \
   -o gpurun_out/$1_full -f python bench.py --steps 3 --warmup 2 --no-e2e --cpu-sample 4 > gpurun_out/$1_full.log 2>&1
echo "$1 rc=$?"
