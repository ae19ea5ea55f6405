"""Per-source-line instruction and stall-sample totals of one ncu report
(development tool).  Usage: python tools/ncu_lines.py REPORT [min_frac]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
res = []
f = None
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            res.append((f, int(r[0]), float(r[7]), float(r[4]), r[1][:100]))
        except ValueError:
            pass
tot = sum(x[2] for x in res) or 1
ts = sum(x[3] for x in res) or 1
print(f"total warp instructions {tot:.4g}, stall samples {ts:.0f}")
for x in sorted(res, key=lambda x: (x[0], x[1])):
    if x[2] / tot > thr or x[3] / ts > thr:
        print(f"{x[0][:12]:12s}:{x[1]:5d} {x[2]/1e6:8.1f}M {x[2]/tot*100:5.1f}% "
              f"stall {x[3]/ts*100:5.1f}%  {x[4]}")
