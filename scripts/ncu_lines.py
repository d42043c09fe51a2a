"""Aggregate an ncu source page (--print-source cuda,sass CSV) by CUDA source line.

    ncu -i rep --page source --csv --kernel-name regex:K --print-source cuda,sass > s.csv
    python scripts/ncu_lines.py s.csv [top]
Prints file:line, warp-instructions executed, stall samples, shared wavefronts
(+ excess) per source line, sorted by stall samples.
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, 0, 0, ""])
cur_file, cur_line, hdr = None, None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 10:
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0]), r[1][:90])
        continue
    if r[2] in ("...", "-"):
        continue
    try:
        samp = int(r[4])
        inst = int(r[7])
        wf = int(r[hdr.index("L1 Wavefronts Shared")] or 0)
        wfx = int(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[cur_line]
    a[0] += inst; a[1] += samp; a[2] += wf; a[3] += wfx
tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
print(f"total warp-inst {tot_i:.4g}  stall samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:<5} inst {v[0]:>11,} ({100*v[0]/tot_i:4.1f}%)  samp {v[1]:>6} ({100*v[1]/tot_s:4.1f}%)  wf {v[2]:>10,} x{v[3]:>10,}  | {k[2]}")
