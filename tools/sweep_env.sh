# Plan-parameter sweep on c3 (profiling aid): one quick_time line per setting.
cd /root/repo
for cfg in "" "PT_CHAIN_BOOST=1000" "PT_CHAIN_BOOST=1000 PT_SIM_SLOTS=2" "PT_SIM_SLOTS=2" "PT_TASK_US=4" "PT_CHAIN_BOOST=1000 PT_TASK_US=4" "PT_CTA_GBS=12"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/quick_time.py c3 2>&1 | grep -v Warn | tail -1 | cut -c1-140
done
