"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle on the same inputs.

Bar (BASELINE.json north_star): fp64 operator / smoother within 1e-12 relative, fp32 path within 1e-5,
Krylov iteration counts equal +-1.
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2410_09497_b200 as smg  # noqa: E402


def rand_vec(k, level, seed, zero_constrained=True):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1.0, 1.0, oracle.sizes(k, level)[4])
    if zero_constrained:
        mask = constrained_mask(k, level)
        x[mask] = 0.0
    return x


def constrained_mask(k, level):
    return oracle.constrained_mask(k, level)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(x, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


# levels >= 2-3 take the TMA staging path with interior bricks; small levels the cp.async path
@pytest.mark.parametrize("k,level", [(1, 0), (1, 1), (1, 2), (1, 3), (1, 4), (2, 0), (2, 1), (2, 2), (2, 3), (2, 4),
                                     (3, 1), (3, 2), (3, 3), (4, 1), (4, 2), (5, 1), (5, 2), (6, 1), (6, 2), (7, 1),
                                     (7, 2)])
def test_vmult_fp64_matches_oracle(k, level):
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 1, zero_constrained=False)  # constrained entries must be ignored
    y_ref = oracle.apply_stokes(k, level, x)
    y = ctx.apply_stokes(level, dev(x)).cpu().numpy()
    assert rel(y, y_ref) <= 1e-12


@pytest.mark.parametrize("k,level", [(1, 2), (1, 3), (2, 2), (2, 3), (3, 1), (3, 2), (4, 2), (5, 2), (7, 2)])
def test_vmult_fp32_matches_oracle(k, level):
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 2)
    y_ref = oracle.apply_stokes(k, level, x)
    y = ctx.apply_stokes(level, dev(x, torch.float32)).double().cpu().numpy()
    assert rel(y, y_ref) <= 1e-5


@pytest.mark.parametrize("k,level", [(1, 2), (2, 1), (2, 3), (3, 2)])
def test_residual(k, level):
    ctx = smg.Context(k, level)
    x, b = rand_vec(k, level, 3), rand_vec(k, level, 4)
    r_ref = oracle.residual(k, level, b, x)
    r = ctx.residual(level, dev(b), dev(x)).cpu().numpy()
    assert rel(r, r_ref) <= 1e-12


@pytest.mark.parametrize("k,level", [(1, 1), (1, 2), (2, 1), (2, 2), (3, 1), (4, 1)])
def test_smoother_fp64_fixed_cg_matches_oracle(k, level):
    # parity mode: a fixed number of inner CG iterations on both sides
    ctx = smg.Context(k, level, cg_max_iter=12, cg_fixed=True, cg_precond=1)
    x0, b = rand_vec(k, level, 5), rand_vec(k, level, 6)
    x_ref, _ = oracle.smooth(k, level, x0, b, oracle.cg_opts(12, 0.0, True, 1))
    x = dev(x0)
    ctx.smooth(level, x, dev(b))
    assert rel(x.cpu().numpy(), x_ref) <= 1e-11


@pytest.mark.parametrize("k,level", [(1, 2), (2, 1)])
def test_smoother_fp32_matches_oracle(k, level):
    ctx = smg.Context(k, level, cg_max_iter=12, cg_fixed=True, cg_precond=1)
    x0, b = rand_vec(k, level, 7), rand_vec(k, level, 8)
    x_ref, _ = oracle.smooth(k, level, x0, b, oracle.cg_opts(12, 0.0, True, 1))
    x = dev(x0, torch.float32)
    ctx.smooth(level, x, dev(b, torch.float32))
    assert rel(x.double().cpu().numpy(), x_ref) <= 1e-4


@pytest.mark.parametrize("k,level", [(1, 1), (2, 1), (2, 2), (3, 1), (4, 1), (5, 1), (7, 1)])
def test_transfer_matches_oracle(k, level):
    ctx = smg.Context(k, level)
    xc = rand_vec(k, level - 1, 9)
    xf = rand_vec(k, level, 10)
    ref_p = oracle.prolongate_add(k, level - 1, xc, xf)
    got = dev(xf)
    ctx.prolongate_add(level - 1, got, dev(xc))
    assert rel(got.cpu().numpy(), ref_p) <= 1e-13
    ref_r = oracle.restrict(k, level - 1, xf)
    got_r = ctx.restrict(level - 1, dev(xf)).cpu().numpy()
    assert rel(got_r, ref_r) <= 1e-13


@pytest.mark.parametrize("k", [1, 2, 3])
def test_coarse_solve_matches_oracle(k):
    ctx = smg.Context(k, 1)
    b = oracle.apply_stokes(k, 0, rand_vec(k, 0, 11))
    ref = oracle.coarse_solve(k, b)
    got = ctx.coarse_solve(dev(b)).cpu().numpy()
    assert rel(got, ref) <= 1e-10


@pytest.mark.parametrize("k,level", [(1, 2), (2, 1)])
def test_vcycle_fp64_matches_oracle(k, level):
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    b = rand_vec(k, level, 12)
    ref = oracle.vcycle(k, level, b, oracle.cg_opts(10, 0.0, True, 1))
    got = ctx.vcycle(level, dev(b)).cpu().numpy()
    assert rel(got, ref) <= 1e-10


@pytest.mark.parametrize("k,level", [(1, 2), (2, 2), (3, 1)])
def test_solve_iteration_counts(k, level):
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-8, cg_fixed=False)
    b = oracle.apply_stokes(k, level, rand_vec(k, level, 13))
    x_ref, it_ref, _ = oracle.fgmres(k, level, b, 1e-8, 40, oracle.cg_opts(30, 1e-8, False, 1))
    for vp in (smg.F64, smg.F32):
        x, it, hist = ctx.solve(level, dev(b), 1e-8, 40, vp)
        assert abs(it - it_ref) <= 1, (vp, it, it_ref)
        xr = x.cpu().numpy()
        res = np.linalg.norm(b - oracle.apply_stokes(k, level, xr)) / np.linalg.norm(b)
        assert res <= 2e-8


@pytest.mark.parametrize("k,level", [(1, 2), (2, 2), (3, 1), (1, 4), (2, 3)])
def test_vmult_host_blockvector_path(k, level):
    # reference-facing path: BlockVector blocks with the cell-local pressure numbering
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 14)
    ys = ctx.vmult_host(level, smg.to_blockvector(x, k, level))
    assert rel(smg.from_blockvector(ys, k, level), oracle.apply_stokes(k, level, x)) <= 1e-12
    ys32 = ctx.vmult_host(level, [b.astype(np.float32) for b in smg.to_blockvector(x, k, level)], smg.F32)
    assert rel(smg.from_blockvector(ys32, k, level).astype(np.float64), oracle.apply_stokes(k, level, x)) <= 1e-5


def test_vec_upload_download_roundtrip():
    k, level = 2, 2
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 15)
    blocks = smg.to_blockvector(x, k, level)
    v = ctx.upload(level, blocks)
    assert np.array_equal(v.cpu().numpy(), x)  # device layout: pressure global lexicographic
    back = ctx.download(level, v)
    for a, b in zip(back, blocks):
        assert np.array_equal(a, b)


def _zero_constrained_(v, k, level):
    """zero the constrained boundary-normal planes of a device level vector in place."""
    n = (2 << level) * (k + 1)
    off = 0
    for c in range(3):
        d = [n, n, n]
        d[c] = n + 1
        blk = v[off:off + d[0] * d[1] * d[2]].view(d[2], d[1], d[0])
        idx = [slice(None)] * 3
        for pl in (0, n):
            idx[2 - c] = pl
            blk[tuple(idx)] = 0
        off += d[0] * d[1] * d[2]


@pytest.mark.parametrize("k,level", [(3, 6), (1, 6)])
def test_c3_size_properties(k, level):
    # C3 (k=3, 128^3, 538 M DoF): symmetry <Ax, y> = <x, Ay>, linearity and zero constrained rows at
    # full size, where the oracle is too slow (SURVEY.md §8(c) size-independent properties)
    ctx = smg.Context(k, level)
    n_ = ctx.sizes(level)[4]
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(n_, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y = torch.rand(n_, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    _zero_constrained_(x, k, level)
    _zero_constrained_(y, k, level)
    Ax = ctx.apply_stokes(level, x)
    a = float(torch.dot(Ax, y))
    Ay = ctx.apply_stokes(level, y)
    b = float(torch.dot(x, Ay))
    assert abs(a - b) <= 1e-10 * max(abs(a), 1.0)
    del Ay
    A2 = ctx.apply_stokes(level, 0.5 * x + y)
    A2 -= 0.5 * Ax
    A2 -= ctx.apply_stokes(level, y)
    assert float(A2.abs().max()) <= 1e-11 * float(Ax.abs().max())
    mask = torch.ones_like(x)
    _zero_constrained_(mask, k, level)
    assert bool((Ax[mask == 0] == 0).all())  # constrained boundary-normal rows are zero


def test_large_level_properties_symmetry_linearity():
    # full-size properties where the oracle is too slow: <A x, y> = <x, A y>, A(ax + y) = aAx + Ay
    k, level = 2, 5
    ctx = smg.Context(k, level)
    n = ctx.sizes(level)[4]
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    mask = torch.from_numpy(constrained_mask(k, level)).cuda()
    x[mask] = 0
    y[mask] = 0
    Ax, Ay = ctx.apply_stokes(level, x), ctx.apply_stokes(level, y)
    a, b = float(torch.dot(Ax, y)), float(torch.dot(x, Ay))
    assert abs(a - b) <= 1e-11 * max(abs(a), 1.0) * 1e3
    A2 = ctx.apply_stokes(level, 0.5 * x + y)
    assert float((A2 - (0.5 * Ax + Ay)).abs().max()) <= 1e-12 * float(Ax.abs().max()) * 10
    assert bool((Ax[mask] == 0).all())


def test_errors_are_loud():
    with pytest.raises(ValueError):
        smg.Context(0, 2)
    ctx = smg.Context(1, 1)
    with pytest.raises(ValueError):
        ctx.apply_stokes(1, torch.zeros(5, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        ctx.apply_stokes(3, ctx.new_vector(1))


# ---- z-slab operator (multi-GPU partition) on virtual slabs of one device ----
@pytest.mark.parametrize("k,level,nslab", [(1, 3, 2), (2, 3, 2), (2, 3, 4), (3, 3, 4), (2, 4, 3), (4, 2, 2), (5, 2, 4)])
def test_slab_vmult_matches_global(k, level, nslab):
    from paper_2410_09497_b200 import slab
    ctx = smg.Context(k, level)
    x = dev(rand_vec(k, level, 16, zero_constrained=False))
    b = dev(rand_vec(k, level, 17))
    y_ref = ctx.apply_stokes(level, x)
    r_ref = ctx.residual(level, b, x)
    bounds = slab.partition(level, nslab)
    lays = [slab.SlabLayout(k, level, z0, z1) for z0, z1 in bounds]
    # ghost layers through the exchange: slabs start with their owned rows only
    xs = []
    for L in lays:
        full = L.extract(x)
        v = torch.zeros_like(full)
        for c in range(4):
            a, bb = L.owned_planes(c)
            L.block(v, c)[a:bb] = L.block(full, c)[a:bb]
        xs.append(v)
    slab.exchange_local(lays, xs)
    y = torch.zeros_like(x)
    r = torch.zeros_like(x)
    dots = 0.0
    for (z0, z1), L, xv in zip(bounds, lays, xs):
        op = slab.SlabOperator(ctx, level, z0, z1)
        yv = op.new_vector()
        op.vmult(yv, xv)
        L.insert_owned(y, yv)
        rv = op.new_vector()
        op.residual(rv, L.extract(b), xv, exchange=False)
        L.insert_owned(r, rv)
        dots += op.dot(yv, yv)
    assert rel(y.cpu().numpy(), y_ref.cpu().numpy()) <= 1e-14
    assert rel(r.cpu().numpy(), r_ref.cpu().numpy()) <= 1e-14
    assert abs(dots - float(torch.dot(y_ref, y_ref))) <= 1e-12 * float(torch.dot(y_ref, y_ref))
    # fp32
    x32 = x.float()
    y32 = torch.zeros_like(x32)
    for (z0, z1), L in zip(bounds, lays):
        op = slab.SlabOperator(ctx, level, z0, z1)
        yv = op.new_vector(torch.float32)
        op.vmult(yv, L.extract(x32), exchange=False)
        L.insert_owned(y32, yv)
    assert rel(y32.double().cpu().numpy(), ctx.apply_stokes(level, x32).double().cpu().numpy()) <= 1e-6


def test_slab_rejects_bad_ranges():
    import ctypes
    ctx = smg.Context(1, 3)
    x = torch.zeros(10 ** 6, dtype=torch.float64, device="cuda")
    # rows of cells [4, 8) need the held range to cover cells 3 .. 8
    rc = smg.lib().smg_residual_held(ctx._h, 3, smg.F64, ctypes.c_void_p(x.data_ptr()), None,
                                     ctypes.c_void_p(x[10:].data_ptr()), 4, 8, 4, 8)
    assert rc == smg.SMG_EINVAL


@pytest.mark.parametrize("k,level,nparts", [(2, 4, 2), (1, 4, 2), (2, 4, 4), (3, 3, 2)])
def test_slab_multigrid_matches_single_gpu(k, level, nparts):
    # distributed V-cycle / FGMRES on virtual slabs (ghost exchange, face patches computed on both
    # sides, restriction from the extended residual, agglomerated coarse levels) == single GPU
    from paper_2410_09497_b200 import slab_mg
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    mg = slab_mg.virtual_partition(ctx, level, nparts)
    assert mg.la < level
    b = dev(rand_vec(k, level, 21))
    for dt in (torch.float64, torch.float32):
        bb = b.to(dt)
        ref = ctx.vcycle(level, bb)
        parts = {p: mg.slabs[p][level].extract(bb) for p in mg.parts}
        xs = mg.vcycle(level, parts, dt)
        got = torch.zeros_like(bb)
        for p in mg.parts:
            mg.slabs[p][level].add_owned_into(got, xs[p])
        tol = 1e-12 if dt == torch.float64 else 1e-5
        assert rel(got.double().cpu().numpy(), ref.double().cpu().numpy()) <= tol
    rhs = ctx.apply_stokes(level, b)
    x_ref, it_ref, _ = ctx.solve(level, rhs, 1e-8, 40, smg.F32)
    parts = {p: mg.slabs[p][level].extract(rhs) for p in mg.parts}
    xs, it, hist = mg.solve(parts, 1e-8, 40, smg.F32)
    assert abs(it - it_ref) <= 1
    got = torch.zeros_like(rhs)
    for p in mg.parts:
        mg.slabs[p][level].add_owned_into(got, xs[p])
    res = float((rhs - ctx.apply_stokes(level, got)).norm() / rhs.norm())
    assert res <= 2e-8
    # same solution as smg_solve, including the mass-weighted pressure mean (both remove it)
    assert rel(got.cpu().numpy(), x_ref.cpu().numpy()) <= 1e-6


def test_cp_async_staging_path_matches_oracle():
    # the cp.async (LDGSTS) staging fallback (SMG_NO_TMA, read once per process) against the oracle,
    # whole-level and slab operator, in a fresh interpreter
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, oracle
import paper_2410_09497_b200 as smg
from paper_2410_09497_b200 import slab
worst = 0.0
for k, level in ((1, 3), (2, 3), (3, 2)):
    ctx = smg.Context(k, level)
    x = np.random.default_rng(3).uniform(-1, 1, oracle.sizes(k, level)[4])
    ref = oracle.apply_stokes(k, level, x)
    xd = torch.from_numpy(x).cuda()
    y = ctx.apply_stokes(level, xd).cpu().numpy()
    worst = max(worst, np.abs(y - ref).max() / np.abs(ref).max())
    got = torch.zeros_like(xd)
    for z0, z1 in slab.partition(level, 2):
        op = slab.SlabOperator(ctx, level, z0, z1)
        yv = op.new_vector()
        op.vmult(yv, op.lay.extract(xd), exchange=False)
        op.lay.insert_owned(got, yv)
    worst = max(worst, np.abs(got.cpu().numpy() - ref).max() / np.abs(ref).max())
print(worst)
'''
    env = dict(os.environ, SMG_NO_TMA="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert out.returncode == 0, out.stderr
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("chunks", ["4", "3", "2", "8", "16"])
def test_vmult_host_pipeline_chunkings(chunks, monkeypatch):
    # the host pipeline overlaps z-chunk copies with the operator rows of the resident chunks: every
    # chunking (SMG_HOST_CHUNKS, read per call) must give the device operator's result
    k, level = 2, 4
    monkeypatch.setenv("SMG_HOST_CHUNKS", chunks)
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 21)
    y_dev = ctx.apply_stokes(level, torch.from_numpy(x).cuda()).cpu().numpy()
    ys = ctx.vmult_host(level, smg.to_blockvector(x, k, level))
    assert rel(smg.from_blockvector(ys, k, level), y_dev) <= 1e-14
    if chunks == "4":
        assert rel(smg.from_blockvector(ys, k, level), oracle.apply_stokes(k, level, x)) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("k,dtype,tol", [(5, "f64", 1e-12), (6, "f64", 1e-12), (7, "f64", 1e-12), (5, "f32", 1e-5),
                                         (7, "f32", 1e-5)])
def test_vmult_high_degree_tma_path_matches_oracle(k, dtype, tol):
    # level 3 (8^3 cells) is the smallest level whose boxes take the TMA staging path at k >= 5 (level <= 2
    # runs the cp.async fallback): the persistent multi-brick pipeline at high degree against the oracle
    level = 3
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 5)
    y_ref = oracle.apply_stokes(k, level, x)
    t = torch.float64 if dtype == "f64" else torch.float32
    y = ctx.apply_stokes(level, dev(x, t)).double().cpu().numpy()
    assert rel(y, y_ref) <= tol
