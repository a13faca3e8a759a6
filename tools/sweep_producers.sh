# Task-slot count sweep on c3 (profiling aid): libpt_b200_p{3,4}.so are built
# with -DPT_EXEC_PRODUCERS=3/4; one quick_time line per library / stage count.
cd /root/repo
python -c "import sys; sys.path.insert(0,'.'); from paper_1410_5910_b200.offline.build import ensure_case; ensure_case('c3')"
for lib in libpt_b200.so libpt_b200_p3.so libpt_b200_p4.so; do
  echo "== $lib parity"
  PT_B200_LIB=paper_1410_5910_b200/$lib timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -1
  for st in "PT_STAGES=3" "PT_STAGES=2" "PT_STAGES=4"; do
    echo "== $lib $st"
    env $st PT_B200_LIB=paper_1410_5910_b200/$lib timeout 300 python tools/quick_time.py c3 2>&1 | grep -v Warn | tail -2 | cut -c1-300
  done
done
