"""Per-opcode instruction / shared-wavefront / stall breakdown of one
.ncu-rep (source page, SASS).  python tools/ncu_ops.py rep [units]
units = number of work units to normalise by (e.g. warp-slices)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: h.index(k) for k in ["Source", "Instructions Executed", "L1 Wavefronts Shared",
                              "L1 Wavefronts Shared Ideal", "Warp Stall Sampling (All Samples)"]}
agg = defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
tot = 0.0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[ix["Source"]].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    base = op.split(".")[0]
    key = op if base in ("LDS", "STS", "LDG", "STG", "LDCU", "LDC") else base
    try:
        v = [float(r[ix[k]] or 0) for k in ["Instructions Executed", "L1 Wavefronts Shared",
                                             "L1 Wavefronts Shared Ideal", "Warp Stall Sampling (All Samples)"]]
    except ValueError:
        continue
    a = agg[key]
    for q in range(4):
        a[q] += v[q]
    tot += v[3]
print(f"{'op':16s} {'inst/u':>9s} {'wf/u':>8s} {'ideal/u':>8s} {'stall%':>7s}")
for op, (ie, wf, wi, st) in sorted(agg.items(), key=lambda x: -x[1][3])[:22]:
    print(f"{op:16s} {ie / units:9.2f} {wf / units:8.2f} {wi / units:8.2f} {100 * st / max(tot, 1):7.1f}")
t = [sum(a[q] for a in agg.values()) for q in range(3)]
print(f"{'TOTAL':16s} {t[0] / units:9.2f} {t[1] / units:8.2f} {t[2] / units:8.2f}")
