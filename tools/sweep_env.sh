# Executor-knob sweep on c3 (profiling aid): one quick_time line per setting.
#   bash tools/sweep_env.sh "PT_POLL_STAGGER=0" "PT_POLL_STAGGER=200" ...
cd /root/repo
python -c "import sys; sys.path.insert(0,'.'); from paper_1410_5910_b200.offline.build import ensure_case; ensure_case('${CASE:-c3}')"
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/quick_time.py ${CASE:-c3} 2>&1 | grep -v Warn | tail -1 | cut -c1-230
done
