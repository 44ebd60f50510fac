"""GPU parity at the configurations the bench and the solves actually run (VERDICT r1 "what's weak" 1-2).

The kernel variants that only appear on fine levels are covered here against the CPU oracle at the
north_star tolerances (BASELINE.json: operator / smoother 1e-12 relative in fp64, 1e-5 in the fp32
multigrid path; Krylov iteration counts +-1):
  * smoother: the warp-per-patch variant (GS = 32, a colour with >= 1184 patches: level >= 4) and the
    4-warp variant (GS = 128, level 3), fixed inner-CG iteration count on both sides;
  * C1 (k = 1, L = 3) V-cycle and MG-FGMRES: iteration count, solution and pressure mean;
  * C2 (k = 2, L = 5) operator apply in fp64 and fp32;
  * BLAS-1 and project_zero_mean at the boundary (block_vector.hpp:52-93, SPEC.md:212-220 KATs);
  * held-slab restriction with the minimal held range (fine cells from 2 c0 - 2).
The C2 MG-FGMRES comparison against the oracle takes minutes of CPU time; it is marked slow and runs
when SMG_SLOW=1 (profiles/r02 keeps its log).
"""
import os

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
        x[oracle.constrained_mask(k, level)] = 0.0
    return x


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(x, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


def weighted_pressure_mean(k, level, x):
    w1 = smg.pressure_node_weights(k)
    s = oracle.sizes(k, level)
    n = (2 << level) * (k + 1)
    p = x[s[0] + s[1] + s[2]:].reshape(n, n, n)
    w = w1[np.arange(n) % (k + 1)]
    return float(np.einsum("zyx,z,y,x->", p, w, w, w) / (w1.sum() ** 3 * (2 << level) ** 3))


# ---- smoother at the fine-level variants ----
@pytest.mark.parametrize("k,level", [(1, 3), (2, 3), (1, 4), (2, 4), (3, 4)])
def test_smoother_fp64_fine_level_variants(k, level):
    # level 3: 343-512 patches per colour -> GS = 128; level 4: 3375-4096 -> GS = 32 (warp per patch)
    ctx = smg.Context(k, level, cg_max_iter=8, cg_fixed=True, cg_precond=1)
    x0, b = rand_vec(k, level, 31), rand_vec(k, level, 32)
    x_ref, _ = oracle.smooth(k, level, x0, b, oracle.cg_opts(8, 0.0, True, 1))
    x = dev(x0)
    ctx.smooth(level, x, dev(b))
    assert rel(x.cpu().numpy(), x_ref) <= 1e-12


@pytest.mark.parametrize("k,level", [(1, 1), (2, 2), (1, 3), (2, 3), (1, 4), (2, 4)])
def test_smoother_fp32_fine_level_variants(k, level):
    # the fp32 V-cycle smoother against the fp64 oracle on the same inputs (north_star: 1e-5)
    ctx = smg.Context(k, level, cg_max_iter=8, cg_fixed=True, cg_precond=1)
    x0, b = rand_vec(k, level, 33), rand_vec(k, level, 34)
    x_ref, _ = oracle.smooth(k, level, x0, b, oracle.cg_opts(8, 0.0, True, 1))
    x = dev(x0, torch.float32)
    ctx.smooth(level, x, dev(b, torch.float32))
    assert rel(x.double().cpu().numpy(), x_ref) <= 1e-5


@pytest.mark.parametrize("k,level", [(1, 1), (2, 1), (3, 1), (4, 1)])
def test_smoother_fp64_coarse_variant_tight(k, level):
    # the 8-warp variant (GS = 256) at the north_star tolerance
    ctx = smg.Context(k, level, cg_max_iter=12, cg_fixed=True, cg_precond=1)
    x0, b = rand_vec(k, level, 35), rand_vec(k, level, 36)
    x_ref, _ = oracle.smooth(k, level, x0, b, oracle.cg_opts(12, 0.0, True, 1))
    x = dev(x0)
    ctx.smooth(level, x, dev(b))
    assert rel(x.cpu().numpy(), x_ref) <= 1e-12


# ---- C1: V-cycle and MG-FGMRES ----
def test_c1_vcycle_fp64_matches_oracle():
    k, level = 1, 3
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    b = rand_vec(k, level, 37)
    ref = oracle.vcycle(k, level, b, oracle.cg_opts(10, 0.0, True, 1))
    got = ctx.vcycle(level, dev(b)).cpu().numpy()
    assert rel(got, ref) <= 1e-11


def test_c1_vcycle_fp32_matches_oracle():
    k, level = 1, 3
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    b = rand_vec(k, level, 38)
    ref = oracle.vcycle(k, level, b, oracle.cg_opts(10, 0.0, True, 1))
    got = ctx.vcycle(level, dev(b, torch.float32)).double().cpu().numpy()
    assert rel(got, ref) <= 1e-5


def _solve_parity(k, level, seed, tol_x):
    # identical preconditioners on both sides (fixed inner CG, fp64 V-cycle): the FGMRES iterates agree,
    # so the iteration count must be equal and x equal to near rounding
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    b = oracle.apply_stokes(k, level, rand_vec(k, level, seed))
    opts = oracle.cg_opts(10, 0.0, True, 1)
    x_ref, it_ref, _ = oracle.fgmres(k, level, b, 1e-8, 40, opts)
    x, it, _ = ctx.solve(level, dev(b), 1e-8, 40, smg.F64)
    x = x.cpu().numpy()
    assert abs(it - it_ref) <= 1, (it, it_ref)
    assert rel(x, x_ref) <= tol_x
    assert abs(weighted_pressure_mean(k, level, x)) <= 1e-13 * max(np.abs(x).max(), 1.0)
    # mixed precision (fp32 V-cycle, the production path): iteration count +-1 and converged
    x32, it32, _ = ctx.solve(level, dev(b), 1e-8, 40, smg.F32)
    assert abs(it32 - it_ref) <= 1, (it32, it_ref)
    x32 = x32.cpu().numpy()
    res = np.linalg.norm(b - oracle.apply_stokes(k, level, x32)) / np.linalg.norm(b)
    assert res <= 1e-8 * 1.5
    return it, it_ref


def test_c1_fgmres_iterations_solution_mean():
    _solve_parity(1, 3, 39, 1e-9)


@pytest.mark.skipif(os.environ.get("SMG_SLOW") != "1", reason="C2 oracle solve takes minutes (SMG_SLOW=1)")
def test_c2_fgmres_iterations_solution_mean():
    _solve_parity(2, 5, 40, 1e-8)


# ---- C2 operator apply ----
@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 1e-5)])
def test_c2_vmult_matches_oracle(dtype, tol):
    k, level = 2, 5
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 41, zero_constrained=False)
    y_ref = oracle.apply_stokes(k, level, x)
    y = ctx.apply_stokes(level, dev(x, dtype)).double().cpu().numpy()
    assert rel(y, y_ref) <= tol


def test_c2_residual_matches_oracle():
    k, level = 2, 5
    ctx = smg.Context(k, level)
    x, b = rand_vec(k, level, 42), rand_vec(k, level, 43)
    r_ref = oracle.residual(k, level, b, x)
    r = ctx.residual(level, dev(b), dev(x)).cpu().numpy()
    assert rel(r, r_ref) <= 1e-12


# ---- BLAS-1 and project_zero_mean (block_vector.hpp:52-93) ----
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_blas1_matches_reference_semantics(dtype):
    k, level = 2, 3
    ctx = smg.Context(k, level)
    a, b = rand_vec(k, level, 44, False), rand_vec(k, level, 45, False)
    da, db = dev(a, dtype), dev(b, dtype)
    an, bn = da.double().cpu().numpy(), db.double().cpu().numpy()
    # dot / norm accumulate in double (block_vector.hpp:53-61)
    assert abs(ctx.dot(level, da, db) - float(an @ bn)) <= 1e-13 * np.abs(an * bn).sum()
    assert abs(ctx.norm(level, da) - float(np.sqrt(an @ an))) <= 1e-13 * np.sqrt(an @ an)
    eps = 1e-15 if dtype == torch.float64 else 1e-7
    y = db.clone()
    ctx.axpy(level, 0.375, da, y)
    assert rel(y.double().cpu().numpy(), bn + 0.375 * an) <= 4 * eps
    y = da.clone()
    ctx.scale(level, -1.25, y)
    assert rel(y.double().cpu().numpy(), -1.25 * an) <= eps
    y = da.clone()
    ctx.subtract_from(level, db, y)
    assert rel(y.double().cpu().numpy(), bn - an) <= 4 * eps


@pytest.mark.parametrize("k,level", [(1, 2), (2, 3), (3, 2)])
def test_project_zero_mean_matches_oracle_and_kats(k, level):
    ctx = smg.Context(k, level)
    x = rand_vec(k, level, 46) + 0.7
    ref = oracle.project_zero_mean(k, level, x)
    got = ctx.project_zero_mean(level, dev(x)).cpu().numpy()
    # the weighted sums differ only in summation order (fp64 tree on the GPU, serial in the oracle)
    assert rel(got, ref) <= 1e-12
    # velocity untouched
    np_ = oracle.sizes(k, level)[3]
    assert np.array_equal(got[:-np_], x[:-np_])
    # KATs: mean of the output 0 to 1e-14; idempotent to 1e-14; constant -> 0
    assert abs(weighted_pressure_mean(k, level, got)) <= 1e-14
    again = ctx.project_zero_mean(level, dev(got)).cpu().numpy()
    assert np.abs(again - got).max() <= 1e-14
    c = np.zeros_like(x)
    c[-np_:] = 3.25
    assert np.abs(ctx.project_zero_mean(level, dev(c)).cpu().numpy()).max() <= 1e-14 * 3.25  # relative


# ---- held-slab restriction with the minimal held fine range ----
@pytest.mark.parametrize("k", [1, 2])
def test_restrict_held_minimal_range(k):
    import ctypes
    from paper_2410_09497_b200.slab_mg import LevelSlab
    level = 3
    ctx = smg.Context(k, level)
    rf = dev(rand_vec(k, level, 47))
    full = ctx.restrict(level - 1, rf).cpu().numpy()
    c0, c1 = 2, 6
    fzlo, fzhi = 2 * c0 - 2, 2 * c1  # the documented footprint, nothing more
    F = LevelSlab(k, level, fzlo, fzhi, ghost=0)
    C = LevelSlab(k, level - 1, c0, c1, ghost=0)
    rfh = F.extract(rf).contiguous()
    rch = torch.zeros(C.total, dtype=torch.float64, device="cuda")
    lib = smg.lib()
    rc = lib.smg_restrict_held(ctx._h, level - 1, smg.F64, ctypes.c_void_p(rch.data_ptr()),
                               ctypes.c_void_p(rfh.data_ptr()), F.zlo, F.zhi, C.zlo, C.zhi, c0, c1)
    assert rc == smg.SMG_OK, lib.smg_last_error(ctx._h)
    torch.cuda.synchronize()
    got = torch.zeros(oracle.sizes(k, level - 1)[4], dtype=torch.float64, device="cuda")
    C.add_owned_into(got, rch)
    got = got.cpu().numpy()
    # compare the rows of the coarse cells [c0, c1)
    probe = torch.zeros(C.total, dtype=torch.float64, device="cuda") + 1.0
    pm = torch.zeros_like(torch.from_numpy(got)).cuda()
    C.add_owned_into(pm, probe)
    mask = pm.cpu().numpy() > 0
    assert np.abs(got[mask] - full[mask]).max() <= 1e-13 * np.abs(full).max()
    # one fine cell less than the footprint is rejected
    rc = lib.smg_restrict_held(ctx._h, level - 1, smg.F64, ctypes.c_void_p(rch.data_ptr()),
                               ctypes.c_void_p(rfh.data_ptr()), fzlo + 1, fzhi, C.zlo, C.zhi, c0, c1)
    assert rc == smg.SMG_EINVAL


def test_coarse_solve_k4_device_factorisation():
    # level-0 pseudo-inverse built by the device LU (coarse.cu) at k = 4 (nf = 4300), against the oracle
    k = 4
    ctx = smg.Context(k, 1)
    b = oracle.apply_stokes(k, 0, rand_vec(k, 0, 48))
    ref = oracle.coarse_solve(k, b)
    got = ctx.coarse_solve(dev(b)).cpu().numpy()
    assert rel(got, ref) <= 1e-10


def test_zmarch_operator_opt_in_matches_oracle():
    # the opt-in z-march operator (vmult_zm.cuh, SMG_ZMARCH=1, read once per process) in a fresh
    # interpreter: apply and residual, k = 1, 2, fp64 / fp32
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, oracle
import paper_2410_09497_b200 as smg
worst64 = worst32 = 0.0
for k, level in ((1, 3), (2, 2), (2, 3)):
    ctx = smg.Context(k, level)
    rng = np.random.default_rng(k + 7 * level)
    x = rng.uniform(-1, 1, oracle.sizes(k, level)[4]); b = rng.uniform(-1, 1, x.size)
    y_ref = oracle.apply_stokes(k, level, x)
    r_ref = b - y_ref; r_ref[oracle.constrained_mask(k, level)] = 0.0
    for dt in (torch.float64, torch.float32):
        xd = torch.from_numpy(x).to("cuda", dt)
        y = ctx.apply_stokes(level, xd).double().cpu().numpy()
        r = ctx.residual(level, torch.from_numpy(b).to("cuda", dt), xd).double().cpu().numpy()
        e = max(np.abs(y - y_ref).max() / np.abs(y_ref).max(), np.abs(r - r_ref).max() / np.abs(r_ref).max())
        if dt == torch.float64: worst64 = max(worst64, e)
        else: worst32 = max(worst32, e)
print(worst64, worst32)
'''
    env = dict(os.environ, SMG_ZMARCH="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert out.returncode == 0, out.stderr
    e64, e32 = map(float, out.stdout.strip().splitlines()[-1].split())
    assert e64 <= 1e-12 and e32 <= 1e-5


# ---- high degrees (k = 5..7): one CTA per patch; fp64 up to k = 5 ----
@pytest.mark.parametrize("k,dtype,tol", [(5, torch.float64, 1e-12), (5, torch.float32, 1e-5), (6, torch.float32, 1e-5),
                                         (7, torch.float32, 1e-5)])
def test_smoother_high_degree_matches_oracle(k, dtype, tol):
    level = 1
    ctx = smg.Context(k, level, cg_max_iter=8, cg_fixed=True, cg_precond=1)
    x0, b = rand_vec(k, level, 50), rand_vec(k, level, 51)
    x_ref, _ = oracle.smooth(k, level, x0, b, oracle.cg_opts(8, 0.0, True, 1))
    x = dev(x0, dtype)
    ctx.smooth(level, x, dev(b, dtype))
    assert rel(x.double().cpu().numpy(), x_ref) <= tol


def test_smoother_fp64_k6_refuses():
    ctx = smg.Context(6, 1)
    x = ctx.new_vector(1)
    with pytest.raises(ValueError):
        ctx.smooth(1, x, x.clone())


@pytest.mark.parametrize("k", [5, 7])
def test_mg_fgmres_high_degree_converges(k):
    # MG-FGMRES (fp32 V-cycle) at k = 5 and k = 7, level 2: the device coarse factorisation at
    # nf = 7344 / 17152 and the one-CTA-per-patch smoother; converged residual checked with the oracle
    level = 2
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5)
    b = oracle.apply_stokes(k, level, rand_vec(k, level, 52))
    x, it, hist = ctx.solve(level, dev(b), 1e-8, 30, smg.F32)
    res = np.linalg.norm(b - oracle.apply_stokes(k, level, x.cpu().numpy())) / np.linalg.norm(b)
    assert res <= 1.5e-8 and it <= 8, (it, res)


@pytest.mark.skipif(os.environ.get("SMG_SLOW") != "1", reason="k = 5 oracle coarse pseudo-inverse takes minutes")
def test_fgmres_k5_iterations_match_oracle():
    k, level = 5, 1
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    b = oracle.apply_stokes(k, level, rand_vec(k, level, 53))
    _, it_ref, _ = oracle.fgmres(k, level, b, 1e-8, 30, oracle.cg_opts(10, 0.0, True, 1))
    _, it, _ = ctx.solve(level, dev(b), 1e-8, 30, smg.F64)
    assert abs(it - it_ref) <= 1, (it, it_ref)


# ---- multi-GPU driver behind the C ABI (csrc/dist.cu) ----
def test_dist_single_rank_equals_single_gpu():
    from paper_2410_09497_b200 import dist as sd
    k, level = 2, 3
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    D = sd.DistContext(ctx, 1, 0).init_single()
    b = dev(oracle.apply_stokes(k, level, rand_vec(k, level, 60)))
    x_ref, it_ref, _ = ctx.solve(level, b, 1e-8, 30, smg.F64)
    x, it, _ = D.solve(D.extract(level, b), 1e-8, 30, smg.F64)
    assert it == it_ref
    assert rel(x.cpu().numpy(), x_ref.cpu().numpy()) <= 1e-12
    y = torch.zeros_like(b)
    D.vmult(level, y, b.clone())
    assert rel(y.cpu().numpy(), ctx.apply_stokes(level, b).cpu().numpy()) <= 1e-14


def test_dist_nccl_transport_one_rank():
    # the in-library NCCL transport (dlopen'ed libnccl) with one rank: init, all-reduce, solve
    import torch.distributed as dist
    from paper_2410_09497_b200 import dist as sd
    if not dist.is_initialized():
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29531", rank=0, world_size=1)
    k, level = 1, 3
    ctx = smg.Context(k, level, cg_max_iter=10, cg_fixed=True)
    D = sd.DistContext(ctx, 1, 0).init_nccl()
    b = dev(oracle.apply_stokes(k, level, rand_vec(k, level, 61)))
    x_ref, it_ref, _ = ctx.solve(level, b, 1e-8, 30, smg.F32)
    x, it, _ = D.solve(D.extract(level, b), 1e-8, 30, smg.F32)
    assert abs(it - it_ref) <= 1
    assert rel(x.cpu().numpy(), x_ref.cpu().numpy()) <= 1e-6
    assert abs(D.dot(level, D.extract(level, b), D.extract(level, b)) - float(b @ b)) <= 1e-12 * float(b @ b)


@pytest.mark.parametrize("k,level,world", [(2, 3, 2), (1, 4, 2), (2, 4, 3)])
def test_dist_multi_process_equals_single_gpu(k, level, world):
    # `world` processes on one GPU, gloo transport callbacks: slab operator, slab V-cycle and FGMRES in
    # C++ == the single-GPU results
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29540 + world + 3 * k + level),
           os.path.join(root, "tests", "dist_worker.py"), str(k), str(level)]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=root, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    r = json.loads(lines[-1])
    assert r["vmult_rel"] <= 1e-14
    assert r["f64"]["iters"] == r["f64"]["iters_single"] and r["f64"]["x_rel"] <= 1e-10
    assert abs(r["f32"]["iters"] - r["f32"]["iters_single"]) <= 1 and r["f32"]["x_rel"] <= 1e-6


# ---- fused halo-residual smoother ----
@pytest.mark.parametrize("k,level", [(1, 1), (1, 3), (2, 2), (2, 4), (3, 1), (3, 3)])
def test_fused_halo_residual_smoother_matches_unfused_and_oracle(k, level):
    # the patch kernel evaluates r = b - A x on the patch rows from the patch window of the colour's
    # snapshot; equal to the global residual, so the smoothing step equals the unfused one (one residual
    # launch per colour) to rounding, and the oracle to the north_star tolerance
    x0, b = rand_vec(k, level, 62), rand_vec(k, level, 63)
    out = {}
    for fused in (False, True):
        ctx = smg.Context(k, level, cg_max_iter=8, cg_fixed=True, cg_precond=1, smoother_fused=fused)
        x = dev(x0)
        ctx.smooth(level, x, dev(b))
        out[fused] = x.cpu().numpy()
    assert rel(out[True], out[False]) <= 1e-13
    x_ref, _ = oracle.smooth(k, level, x0, b, oracle.cg_opts(8, 0.0, True, 1))
    assert rel(out[True], x_ref) <= 1e-12
    # fp32 path and the full solve with the fused smoother
    ctx = smg.Context(k, level, cg_max_iter=8, cg_fixed=True, cg_precond=1, smoother_fused=True)
    x = dev(x0, torch.float32)
    ctx.smooth(level, x, dev(b, torch.float32))
    assert rel(x.double().cpu().numpy(), x_ref) <= 1e-5


def test_fused_smoother_solve_iterations():
    k, level = 2, 3
    b = dev(oracle.apply_stokes(k, level, rand_vec(k, level, 64)))
    its = {}
    for fused in (False, True):
        ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5, smoother_fused=fused)
        _, its[fused], _ = ctx.solve(level, b, 1e-8, 30, smg.F32)
    assert abs(its[True] - its[False]) <= 1


def test_graph_captured_vcycle_survives_tensor_map_recycling():
    # the solve replays a captured V-cycle whose kernels hold tensor-map slot addresses: recycling the
    # other slots (70 applies on distinct vectors) must not change the next solve
    k, level = 2, 3
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-5)
    b = dev(oracle.apply_stokes(k, level, rand_vec(k, level, 65)))
    x1, it1, _ = ctx.solve(level, b, 1e-8, 30, smg.F32)
    vecs = [torch.rand_like(b) for _ in range(70)]
    for v in vecs:
        ctx.apply_stokes(level, v)
    x2, it2, _ = ctx.solve(level, b, 1e-8, 30, smg.F32)
    assert it1 == it2
    assert rel(x2.cpu().numpy(), x1.cpu().numpy()) <= 1e-12
