#!/bin/bash
# Profiling aid: one ncu --set full capture of the executor per program
# (A, M, AM) at the given cases; reports under gpurun_out/.
#   tools/ncu_programs.sh TAG "c3 c2" "A M AM"
TAG=$1; CASES=${2:-c3}; KINDS=${3:-"A M AM"}
mkdir -p gpurun_out
for c in $CASES; do
  python -c "import sys; sys.path.insert(0,'.'); from paper_1410_5910_b200.offline.build import ensure_case; ensure_case('$c')" > /dev/null 2>&1
  for k in $KINDS; do
    ncu --set full --import-source on --clock-control none -k regex:pt_exec_kernel -s 2 -c 1 \
        -f -o gpurun_out/${TAG}_ncu_${c}_${k} python tools/ncu_target.py $c $k 4 > gpurun_out/${TAG}_ncu_${c}_${k}.log 2>&1
    tail -1 gpurun_out/${TAG}_ncu_${c}_${k}.log
  done
done
