"""Warp-stall samples per CUDA source line of one .ncu-rep (needs -lineinfo
and --import-source): python tools/ncu_lines.py rep [top]
Prints the hottest lines with their share of all samples and the top stall
reasons on each line."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    vals = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") or "Stall Sampling (All" in h or h == "Instructions Executed":
            try:
                vals[h] = float(r[i] or 0)
            except ValueError:
                pass
    a = agg.setdefault(key, {"src": r[1][:70]})
    for k, v in vals.items():
        a[k] = a.get(k, 0) + v
S = "Warp Stall Sampling (All Samples)"
tot = sum(a.get(S, 0) for a in agg.values()) or 1
stall_cols = sorted({k for a in agg.values() for k in a if k not in (S, "src", "Instructions Executed")})
for key, a in sorted(agg.items(), key=lambda kv: -kv[1].get(S, 0))[:top]:
    reasons = sorted(((a.get(c, 0), c) for c in stall_cols), reverse=True)[:3]
    rs = " ".join(f"{c.replace('stall_', '')}={v / max(a.get(S, 1), 1):.0%}" for v, c in reasons if v)
    print(f"{100 * a.get(S, 0) / tot:5.1f}% {key[0]}:{key[1]:<4} {a['src']:<70} {rs}")
