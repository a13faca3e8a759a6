# Sync-free triangular-solve knobs on c3 (profiling aid): one online_e2e line per setting.
cd /root/repo
python -c "import sys; sys.path.insert(0,'.'); from paper_1410_5910_b200.offline.build import ensure_case; ensure_case('${CASE:-c3}')"
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/online_e2e.py ${CASE:-c3} 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print({k: round(v*1e3,2) for k,v in d['device_stage_seconds'].items()})"
done
