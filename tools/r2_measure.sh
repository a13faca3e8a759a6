#!/bin/bash
# Profiling aid: GPU tests, apply/solve timings and executor traces at c3.
#   tools/r2_measure.sh TAG [pytest-args]
TAG=${1:-run}
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu ${2:-} > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
python tools/quick_time.py c3 c2 c1 > gpurun_out/${TAG}_time.txt 2>&1; grep -v Warn gpurun_out/${TAG}_time.txt | grep "c[0-9]:"
for k in A M AM; do
  python tools/critical_path.py c3 $k --dump gpurun_out/${TAG}_trace_c3_$k.npz > gpurun_out/${TAG}_cp_c3_$k.txt 2>&1
  head -2 gpurun_out/${TAG}_cp_c3_$k.txt
done
