#!/bin/bash
# Round-end evidence on a GPU box: test log, bench lines of every config,
# ncu launch list of the bench and per-program ncu captures (c2).
#   tools/r2_final.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; tail -1 gpurun_out/${TAG}_pytest_gpu.txt
python bench.py > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err; tail -c 400 gpurun_out/${TAG}_bench_c3.json
: > gpurun_out/${TAG}_all_configs.jsonl
for c in c1 c2 c3r c3 c5; do
  python bench.py --config $c --no-cpu-baseline --no-online 2>/dev/null | tail -1 >> gpurun_out/${TAG}_all_configs.jsonl
done
wc -l gpurun_out/${TAG}_all_configs.jsonl
PT_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-online \
  > gpurun_out/${TAG}_ncu_bench.log 2>&1
wc -l gpurun_out/${TAG}_launches_c3.csv
bash tools/ncu_programs.sh ${TAG}t "c2" "A M AM" > gpurun_out/${TAG}_ncu_c2_tiles.log 2>&1; tail -1 gpurun_out/${TAG}_ncu_c2_tiles.log
