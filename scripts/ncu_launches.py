"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel.

    python scripts/ncu_launches.py launches.csv [skip_first_n_launches]
"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
i_k, i_m, i_v, i_id = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
per, names = collections.defaultdict(dict), {}
for r in rows[1:]:
    per[r[i_id]][r[i_m]] = float(r[i_v].replace(",", ""))
    names[r[i_id]] = r[i_k]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for k, v in per.items():
    if int(k) < skip:
        continue
    n = names[k].split("(")[0].split("<")[0].replace("void ", "").replace("rbm::", "")
    a = agg[n]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0.0)
    a[2] += v.get("dram__bytes_read.sum", 0.0)
    a[3] += v.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':28s} {'launches':>8s} {'mean ms':>9s} {'share':>6s} {'read GB':>8s} {'write GB':>9s}")
for n, a in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"{n:28s} {a[0]:8d} {a[1] / a[0] / 1e6:9.3f} {100 * a[1] / tot:5.1f}% {a[2] / a[0] / 1e9:8.3f} {a[3] / a[0] / 1e9:9.3f}")
