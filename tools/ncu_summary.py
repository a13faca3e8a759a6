"""Summaries of ncu output for profiles/ (profiling aid, not product code).

    python tools/ncu_summary.py rep  <file.ncu-rep> <label> [command]   # --set full capture
    python tools/ncu_summary.py list <launches.csv> [command]           # --metrics gpu__time_duration.sum
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic"]


def rep(path, label, command=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, res = rows[0], rows[1], []
    for v in rows[2:]:
        d = OrderedDict(kernel=v[h.index("Kernel Name")])
        for k in KEYS:
            if k in h:
                d[k] = f"{v[h.index(k)]} {units[h.index(k)]}".strip()
        stalls = {n.split("issue_stalled_")[1].replace("_per_issue_active.ratio", ""): float(v[i])
                  for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_")
                  and n.endswith("_per_issue_active.ratio") and v[i] not in ("", "n/a")}
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        try:
            d["traffic_bytes"] = float(v[h.index("dram__bytes_read.sum")]) + \
                float(v[h.index("dram__bytes_write.sum")])
        except ValueError:
            pass
        res.append(d)
    print(json.dumps({"label": label, "command": command, "launches": res}, indent=1))


def launch_list(path, command=None):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    kn, mv, unit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        t = float(r[mv].replace(",", ""))
        u = r[unit]
        t = t / 1e3 if u in ("ns", "nsecond") else (t * 1e3 if u in ("ms", "msecond") else t)
        a = agg.setdefault(r[kn], [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    print(json.dumps({
        "command": command,
        "note": "ncu serialises launches with cold caches (PT_GRAPH=0: ncu does not profile kernels "
                "inside conditional graph bodies); shares, not absolute times, compare with bench.py",
        "launches_profiled": sum(v[0] for v in agg.values()),
        "kernels": {k: {"launches": n, "total_us": round(t, 1), "avg_us": round(t / n, 2),
                        "share": round(t / tot, 4)} for k, (n, t) in agg.items()}}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        rep(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launch_list(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
