"""Instruction mix and stall attribution from an ncu report's SASS source page."""
import csv, subprocess, sys
from collections import Counter
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iS, iW, iI = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(float(r[iW] or 0) for r in rows[2:]); ti = sum(float(r[iI] or 0) for r in rows[2:])
c, ci = Counter(), Counter()
for r in rows[2:]:
    t = r[iS].split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = op.split(".")[0]
    c[op] += float(r[iW] or 0); ci[op] += float(r[iI] or 0)
print(f"samples {tot:.0f} warp-instructions {ti:.4g}")
for op, v in ci.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 22):
    print(f"{op:10s} inst {v / ti * 100:5.1f}%  stall-samples {c[op] / tot * 100:5.1f}%")
sc = Counter()
for r in rows[2:]:
    for i in stall_cols: sc[h[i]] += float(r[i] or 0)
st = sum(sc.values())
print("stalls:", ", ".join(f"{k[6:]} {v / st * 100:.1f}%" for k, v in sc.most_common(8)))
