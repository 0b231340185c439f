"""Best time per (lx, mode) per variant from tools/abn.sh / ab_env.sh output:
python tools/ab_summary.py FILE"""
import collections
import re
import sys

res = collections.defaultdict(lambda: collections.defaultdict(list))
cur = None
order = []
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line.split()[1]
        if cur not in order:
            order.append(cur)
        continue
    m = re.match(r'\{"lx": (\d+), "nel": \d+, "mode": "(\w+)", "ms": ([\d.]+)', line)
    if m:
        res[(int(m.group(1)), m.group(2))][cur].append(float(m.group(3)))
for k in sorted(res):
    base = min(res[k][order[0]]) if res[k][order[0]] else None
    cells = []
    for c in order:
        if res[k][c]:
            v = min(res[k][c])
            cells.append(f"{c.split('/')[-2] if '/' in c else c} {v:.4f}" + (f" ({base / v:.2f}x)" if base else ""))
    print(f"lx={k[0]:2d} {k[1]:6s} " + "  ".join(cells))
