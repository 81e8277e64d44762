#!/usr/bin/env python
"""Source lines of one kernel ranked by warp-stall samples (ncu --import-source report):
  python scripts/ncu_source_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, res = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or r[2] != "-":
        continue
    ie = int(r[hdr.index("Instructions Executed")] or 0)
    samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    res.append((ie, samp, cur, r[0], r[1][:100]))
tot = sum(o[0] for o in res) or 1
ts = sum(o[1] for o in res) or 1
print(f"instructions {tot / 1e6:.1f} M, stall samples {ts}")
for o in sorted(res, key=lambda o: -o[1])[:top]:
    print(f"{o[0] / 1e6:8.1f}M {100 * o[0] / tot:5.1f}% samp {100 * o[1] / ts:5.1f}% {o[2]}:{o[3]} {o[4]}")
