"""Top source lines by warp-stall samples from an ncu report (profiling aid).

    python tools/ncu_lines.py <file.ncu-rep> [n]
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, recs, total = None, None, [], 0
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or r[2] != "-":
            continue
        s = int(r[4] or 0)
        total += s
        stalls = {hdr[i][6:]: int(r[i]) for i in range(len(hdr))
                  if hdr[i].startswith("stall_") and r[i] not in ("", "0") and r[i].isdigit()}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        recs.append((s, fname, r[0], r[1].strip()[:70], top))
    recs.sort(key=lambda t: -t[0])
    print(f"total samples {total}")
    for s, f, ln, src, top in recs[:n]:
        print(f"{100.0 * s / max(total, 1):5.1f}% {f}:{ln:<5} {src:<70} {top}")


if __name__ == "__main__":
    main()
