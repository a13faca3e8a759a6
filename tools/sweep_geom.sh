#!/bin/bash
# Profiling aid: c3 apply / solve timings over executor geometry knobs.
#   tools/sweep_geom.sh TAG "ENV1=.. ENV2=.." "ENV1=.." ...
TAG=$1; shift
mkdir -p gpurun_out
for cfg in "$@"; do
  echo "== $cfg" | tee -a gpurun_out/${TAG}_geom.txt
  env $cfg PT_VERBOSE=1 timeout 90 python tools/quick_time.py c3 2>&1 | grep -v Warn | grep "c[0-9]:\|pt_create\|rror" | tee -a gpurun_out/${TAG}_geom.txt
done
