"""Summarise tools/ab.sh output: best time per (lx, mode) for A and B, B/A.
python tools/ab_table.py FILE  (or the output on stdin: tools/ab.sh ... | python tools/ab_table.py)"""
import collections
import re
import sys

cur = None
res = collections.defaultdict(list)
for line in (open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin):
    if line.startswith("=="):
        cur = line.split()[1]
        continue
    m = re.match(r'\{"lx": (\d+), "nel": \d+, "mode": "(\w+)", "ms": ([\d.]+)', line)
    if m:
        res[(int(m.group(1)), m.group(2), cur)].append(float(m.group(3)))
for k in sorted({(a, b) for a, b, _ in res}):
    A, B = res[(k[0], k[1], "A")], res[(k[0], k[1], "B")]
    if A and B:
        print(f"lx={k[0]:2d} {k[1]:6s} A {min(A):.4f} B {min(B):.4f}  B/A {min(B) / min(A):.3f}")
