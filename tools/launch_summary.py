"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/launch_summary.py launches.csv [header line]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
agg = defaultdict(list)
for r in rows[start + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    agg[r[ix["Kernel Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("(cold-cache, serialised replay: compare SHARES, not absolutes; numbers printed by that run are not bench values)\n")
print("launches    mean us  share  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):8d} {sum(v) / len(v):10.1f} {100 * sum(v) / tot:5.1f}%  {k[:100]}")
