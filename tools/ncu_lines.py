"""Per-source-line attribution of an ncu report's SASS counters (stall samples, instructions, shared
wavefronts) through the line table of the kernel's cubin (nvdisasm -g).
Usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ.o KERNEL_SUBSTRING [RANGES]
RANGES: comma-separated name=first-last line ranges of the source file to bucket (e.g. pass1=520-585)."""
import csv
import collections
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True, check=True)
    cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
    found = []
    for cb in cubins:
        dis = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
        # split per function
        funcs = re.split(r"\n\s*\.text\.(\S+):", dis)
        for i in range(1, len(funcs), 2):
            if kernel_sub in funcs[i]:
                found.append((funcs[i], funcs[i + 1]))
    if len(found) != 1:
        # a substring matching several instantiations would attribute with the wrong line table
        raise SystemExit(f"{len(found)} functions match {kernel_sub!r}: " + ", ".join(n for n, _ in found))
    name, body = found[0]
    table, cur = {}, None
    for ln in body.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return name, table


def main():
    rep, obj, ksub = sys.argv[1:4]
    ranges = []
    if len(sys.argv) > 4:
        for part in sys.argv[4].split(","):
            nm, rg = part.split("=")
            a, b = map(int, rg.split("-"))
            ranges.append((nm, a, b))
    name, table = line_table(obj, ksub)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    iA, iW, iI = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    iSW = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
    stall_cols = {k: i for i, k in enumerate(h) if k.startswith("stall_")}
    base = int(rows[2][iA], 16)
    per = collections.defaultdict(lambda: collections.Counter())
    for r in rows[2:]:
        if len(r) <= iI or not r[iA]:
            continue
        off = int(r[iA], 16) - base
        key = table.get(off, ("?", 0))
        c = per[key]
        c["samples"] += float(r[iW] or 0)
        c["inst"] += float(r[iI] or 0)
        if iSW is not None:
            c["smem_wf"] += float(r[iSW] or 0)
        for k, i in stall_cols.items():
            c[k] += float(r[i] or 0)
    tot = collections.Counter()
    for c in per.values():
        tot.update(c)
    print(f"kernel {name[:90]}\ntotal samples {tot['samples']:.0f} inst {tot['inst']:.4g} smem wavefronts {tot['smem_wf']:.4g}")
    if ranges:
        for nm, a, b in ranges:
            agg = collections.Counter()
            for (f, l), c in per.items():
                if a <= l <= b:
                    agg.update(c)
            top = sorted(((v, k) for k, v in agg.items() if k.startswith("stall_")), reverse=True)[:4]
            tops = " ".join(f"{k[6:]}={v / max(agg['samples'], 1) * 100:.0f}%" for v, k in top)
            print(f"{nm:10s} lines {a}-{b}: samples {agg['samples'] / tot['samples'] * 100:5.1f}%  inst "
                  f"{agg['inst'] / tot['inst'] * 100:5.1f}%  smem {agg['smem_wf'] / max(tot['smem_wf'], 1) * 100:5.1f}%  [{tops}]")
    print("top lines by samples:")
    for (f, l), c in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[:25]:
        print(f"  {f}:{l:<5d} samples {c['samples'] / tot['samples'] * 100:5.1f}%  inst {c['inst'] / tot['inst'] * 100:5.1f}%")


if __name__ == "__main__":
    main()
