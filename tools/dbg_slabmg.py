import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_09497_b200 as smg
from paper_2410_09497_b200 import slab_mg
k, level, nparts = 2, 4, 4
ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
mg = slab_mg.virtual_partition(ctx, level, nparts)
print("la", mg.la, mg.bounds)
x = torch.rand(ctx.sizes(level)[4], dtype=torch.float64, device="cuda")
ref = ctx.apply_stokes(level, x)
parts = {p: mg.slabs[p][level].extract(x) for p in mg.parts}
for p in mg.parts:  # zero the ghosts
    S = mg.slabs[p][level]
    for c in range(4):
        a, b = S.owned_planes(c)
        blk = S.block(parts[p], c)
        blk[:a] = 0
        blk[b:] = 0
mg.exchange(level, parts)
y = {p: torch.zeros_like(parts[p]) for p in mg.parts}
mg.vmult(level, y, parts)
got = torch.zeros_like(x)
for p in mg.parts:
    mg.slabs[p][level].add_owned_into(got, y[p])
print("vmult rel err", float((got - ref).abs().max() / ref.abs().max()))
for p in mg.parts:
    S = mg.slabs[p][level]
    e = S.extract(x)
    for c in range(4):
        d = (S.block(parts[p], c) - S.block(e, c)).abs().max(dim=1).values
        bad = torch.nonzero(d).flatten().tolist()
        if bad: print("part", p, "block", c, "ghost planes differing:", bad[:5], "of", S.planes[c])
b = ctx.apply_stokes(level, torch.rand(ctx.sizes(level)[4], dtype=torch.float64, device="cuda"))
xr, itr, hr = ctx.solve(level, b, 1e-8, 40, smg.F32)
parts = {p: mg.slabs[p][level].extract(b) for p in mg.parts}
xs, it, hist = mg.solve(parts, 1e-8, 40, smg.F32)
print("ref hist", itr, hr)
print("slab hist", it, hist)
got = torch.zeros_like(b)
for p in mg.parts:
    mg.slabs[p][level].add_owned_into(got, xs[p])
print("res", float((b - ctx.apply_stokes(level, got)).norm() / b.norm()))
# V-cycle on a zero-ghost input
v = {p: mg.slabs[p][level].extract(b).float() for p in mg.parts}
for p in mg.parts:
    S = mg.slabs[p][level]
    for c in range(4):
        a, bb = S.owned_planes(c)
        blk = S.block(v[p], c); blk[:a] = 0; blk[bb:] = 0
z = mg.vcycle(level, v, torch.float32)
zr = ctx.vcycle(level, b.float())
got = torch.zeros_like(zr)
for p in mg.parts:
    mg.slabs[p][level].add_owned_into(got, z[p])
print("vcycle zero-ghost input rel err", float((got - zr).abs().max() / zr.abs().max()))
z2 = mg.vcycle(level, v, torch.float32)
got2 = torch.zeros_like(zr)
for p in mg.parts:
    mg.slabs[p][level].add_owned_into(got2, z2[p])
print("second vcycle rel err", float((got2 - zr).abs().max() / zr.abs().max()))
