#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the
# executor, Arnoldi and batched kernels on tiny fixtures; logs under
# gpurun_out/.  Profiling aid.   tools/sanitize.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
FIX="fx_plr fx_uneven fx_l2 fx_extrap_plr fx_extrap"
for tool in memcheck racecheck synccheck initcheck; do
  for graph in 1 0; do
    log=gpurun_out/${TAG}_${tool}_graph${graph}.log
    PT_GRAPH=$graph timeout 1200 compute-sanitizer --tool $tool --print-limit 50 \
        --kernel-name-exclude kns=at::,kns=cutlass,kns=elementwise,kns=reduce \
        python tools/sanitize_driver.py $FIX > $log 2>&1
    echo "$tool graph=$graph rc=$? $(grep -c 'ERROR SUMMARY' $log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | head -2 | tr '\n' ' ')"
  done
done
