"""Benchmark: Stokes operator-apply DoF/s (fp64) on the BASELINE.json workload, with the smoother
(fp32), the MG-FGMRES solve, the end-to-end host-buffer path, the roofline of the dominant kernel and
the CPU baseline on this box's host cores. Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (configs[1] of BASELINE.json, the largest config that fits one GPU and that the metric is
quoted on): 3D unit-cube Stokes, RT_2 velocity / DGQ_2 pressure, 64^3 cells (level 5), 28.4 M DoF.
Each step is one fp64 operator apply y = A x; x and y are 227 MB each (> 126 MB L2), so no L2 flush
is needed between steps. Under torchrun (N > 1) the SAME global problem is split into N z-slabs, one
per GPU (strong scaling): each step is the ghost-layer exchange over NCCL (P2P send/recv of one cell
layer per neighbour and block) followed by the slab operator; value = global DoF / max-over-ranks
step time. The MG solve runs on the same slabs (slab_mg: ghost exchange per smoothing colour, coarse
levels agglomerated) -- all through the C ABI's multi-GPU driver (smg_dist_*, csrc/dist.cu); the smoother
DoF/s line is reported at N = 1 only.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEGREE, LEVEL = 2, 5
FP64_PEAK_TFLOPS = 33.3  # tools/fma_peak.cu on this pool's B200 (profiles/r01/fma_peaks.txt)
FP32_PEAK_TFLOPS = 69.58
METRIC = "Stokes operator-apply DoF/s (fp64), RT_2 64^3 cells; + fp32 smoother DoF/s and MG-FGMRES solve time"


# brick shapes of the operator kernel per degree (fp64), csrc/vmult_kernel.cuh BrickShape
SHAPES = {1: "8x4x4-cell bricks, 2 CTAs/SM, 256 threads", 2: "4x4x4-cell bricks, 1 CTA/SM, 384 threads, two U and two Q buffers, no barrier after pass 3",
          3: "4x2x2-cell bricks, 1 CTA/SM, 256 threads", 4: "2x2x2-cell bricks, 384 threads"}


def dofs(k, level):
    n = (2 << level) * (k + 1)
    return 3 * (n + 1) * n * n + n ** 3


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "20", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region starts only once the sampler is producing lines
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.start = len(self.lines)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.stop = len(self.lines)
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # samples taken while the timed region ran (plus the one right after it, so a short region
        # still has a reading)
        lines = self.lines[getattr(self, "start", 0):getattr(self, "stop", len(self.lines)) + 1]
        for ln in lines:
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)["dram_bytes_per_launch"].get(key)
    except Exception:
        return None


def _oracle_native():
    import oracle
    oracle.use_native()  # -march=native build, compiled on this host (reference Release flags)
    return oracle


def cpu_baseline(k, level, smoke=False):
    """The CPU oracle (restatement of the reference algorithm: Alg. 1 cell/face loops, colour-parallel
    patch smoother; built with the reference's Release flags -O3 -march=native -funroll-loops + OpenMP,
    proj/CMakeLists.txt:26-27) timed on this host's cores, BASELINE.md §5 legs:
      vmult at the benchmarked workload (C2, all threads: the whole level; 1 thread: a z-slab sample),
      the smoothing step at C2 (z-slab samples of patches + their residual rows, all / 1 thread),
      V-cycle at C1 (whole problem, all / 1 thread) and the MG-FGMRES solve at C1 (all threads).
    Samples are z-slabs of the SAME level (identical per-DoF work); DoF/s = DoF in the sample / time."""
    import numpy as np
    oracle = _oracle_native()
    ncpu = os.cpu_count()
    m = 2 << level
    N = dofs(k, level)
    per_layer = N / m
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, N)
    y = np.zeros(N)
    legs = {}

    def timeit(fn, min_s=1.0, max_reps=20):
        fn()  # warm-up (tables, page faults)
        reps, t0 = 0, time.perf_counter()
        while True:
            fn()
            reps += 1
            if time.perf_counter() - t0 >= min_s or reps >= max_reps:
                break
        return (time.perf_counter() - t0) / reps, reps

    for threads in (ncpu, 1):
        oracle.set_threads(threads)
        tag = "all" if threads == ncpu else "1thread"
        nz = m if threads == ncpu else max(2, m // 32)
        if nz == m:
            dt, reps = timeit(lambda: oracle.apply_stokes(k, level, x), 2.0, 5)
        else:
            dt, reps = timeit(lambda: oracle.apply_stokes_sample(k, level, x, 0, nz, y), 1.0, 5)
        legs[f"vmult_C2_{tag}"] = {"dofs_per_s": per_layer * nz / dt, "threads": threads, "reps": reps,
                                   "sample": "whole level" if nz == m else f"cells z in [0,{nz}) of {m}"}
        if smoke:
            continue
        # smoothing step (fp64 oracle; the GPU step is fp32), patches with vertex planes [1, vz1]
        vz1 = 8 if threads == ncpu else 1
        b = oracle.apply_stokes(k, level, x) if threads == ncpu else y
        xs = np.zeros(N)
        opts = oracle.cg_opts(30, 1e-5, False, 1)
        t0 = time.perf_counter()
        oracle.smooth_sample(k, level, xs, b, 1, vz1, opts)
        dt = time.perf_counter() - t0
        legs[f"smooth_C2_{tag}"] = {"dofs_per_s": per_layer * vz1 / dt, "threads": threads, "s_per_sample": dt,
                                    "sample": f"patches with vertex z in [1,{vz1}] + their residual rows "
                                              f"(~{vz1} of {m} cell layers), cg_tol 1e-5"}
        # C1: V-cycle and solve (k=1, level 3), whole problem
        k1, l1 = 1, 3
        n1 = dofs(k1, l1)
        b1 = oracle.apply_stokes(k1, l1, rng.uniform(-1, 1, n1))
        o1 = oracle.cg_opts(30, 1e-8, False, 1)
        dt, reps = timeit(lambda: oracle.vcycle(k1, l1, b1, o1), 0.5, 10)
        legs[f"vcycle_C1_{tag}"] = {"s": dt, "dofs_per_s": n1 / dt, "threads": threads}
        if threads == ncpu:  # (single-threaded: ~20 s, the V-cycle leg gives the 1-thread rate)
            t0 = time.perf_counter()
            _, it, _ = oracle.fgmres(k1, l1, b1, 1e-8, 40, o1)
            dt = time.perf_counter() - t0
            legs[f"solve_C1_{tag}"] = {"s": dt, "iterations": it, "ns_per_dof": dt / n1 * 1e9, "threads": threads}
    oracle.set_threads(ncpu)
    v = legs["vmult_C2_all"]["dofs_per_s"]
    return {"value": v, "unit": "DoF/s", "cores": ncpu, "kind": "port",
            "sample": f"oracle Alg.1 vmult fp64 at k={k}, level {level} ({m}^3 cells, {N} DoF, the benchmarked "
                      f"workload), whole level, OpenMP {ncpu} threads; -O3 -march=native -funroll-loops",
            "legs": legs}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    oracle = _oracle_native()
    k, level = args.degree, args.level
    m = 2 << level
    N = dofs(k, level)
    x = np.random.default_rng(0).uniform(-1, 1, N)
    y = np.zeros(N)
    # one whole-level apply measures the cost; every step is then a z-slab sample of the SAME level
    # (identical per-DoF work) sized so that the --steps run stays within ~90 s
    t0 = time.perf_counter()
    oracle.apply_stokes(k, level, x)
    t_full = time.perf_counter() - t0
    nz = max(1, min(m, int(m * 90.0 / max(args.steps * t_full, 1e-9))))
    for _ in range(args.warmup):
        oracle.apply_stokes_sample(k, level, x, 0, nz, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.apply_stokes_sample(k, level, x, 0, nz, y)
    dt = time.perf_counter() - t0
    n_sample = N * nz / m
    value = n_sample * args.steps / dt
    sample = (f"reference CPU path (oracle restatement of Alg. 1; the reference ships no code for this path), "
              f"vmult fp64 at k={k}, level {level} ({m}^3 cells): each step the cells z in [0,{nz}) of the level "
              f"(~{n_sample:.0f} DoF; whole level {t_full:.2f} s); all {os.cpu_count()} host threads, "
              f"-O3 -march=native -funroll-loops")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(k, level),
        "cpu_baseline": {"value": value, "unit": "DoF/s", "cores": os.cpu_count(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def workload_config(k, level):
    m = 2 << level
    name = {(2, 5): "C2", (3, 6): "C3", (1, 3): "C1"}.get((k, level), "custom")
    n = dofs(k, level)
    return {"workload": f"{name}: 3D unit-cube Stokes RT_{k}/DGQ_{k}, {m}^3 cells (level {level}), fp64 operator apply",
            "degree": k, "level": level, "dofs": n,
            "l2": f"inputs larger than L2 (x, y {8 * n / 1e6:.0f} MB each vs 126 MB L2); no flush" if 8 * n > 126e6
            else "inputs smaller than L2: an L2 flush is NOT applied, numbers are L2-resident"}


def smoother_flops(k, patches, cg_iters):
    """Algorithmic flops of the patch smoother kernel: per inner CG iteration 12 NP NO^3 + 8 NO^4 FMAs (the
    18 contractions of S d = sum_c G_c Lambda_c^-1 G_c^T d plus the 3 of the pressure-mass preconditioner,
    csrc/smoother_kernel.cuh), and the gather / right-hand side / final update counted as 2 iterations."""
    NP, NO = 2 * k + 1, 2 * k + 2
    per_it = 2 * (12 * NP * NO ** 3 + 8 * NO ** 4)
    return per_it * (cg_iters + 2 * patches)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 300 on the GPU arm: a timed region of ~0.1 s, several clock samples; "
                    "100 on the reference arm)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--degree", type=int, default=DEGREE)
    ap.add_argument("--level", type=int, default=LEVEL)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only to test the multi-rank "
                    "logic on a single-GPU box (CPU-staged exchange, timings meaningless)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 300 if args.impl == "b200" else 100
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch

    import paper_2410_09497_b200 as smg

    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(args.dist_backend)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda" if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    k, level = args.degree, args.level
    N = dofs(k, level)
    ctx = smg.Context(k, level, device=local, cg_max_iter=30, cg_tol=1e-5, cg_fixed=False, cg_precond=1)
    g = torch.Generator(device="cuda").manual_seed(1234)
    x = torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, steps, clocks=False):
        for _ in range(args.warmup):
            fn()
        barrier()
        sampler = ClockSampler(local) if clocks else None
        if sampler:
            sampler.__enter__()
        ev0.record(stream)
        for _ in range(steps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        if sampler:
            sampler.__exit__(None, None, None)
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1) / steps), sampler

    extra = {}
    if world == 1:
        # ---- headline: fp64 vmult, inputs resident in HBM ----
        y = torch.empty_like(x)
        l0 = ctx.launch_count
        ms, clk = timed(lambda: ctx.apply_stokes(level, x, out=y), args.steps, clocks=True)
        launches = (ctx.launch_count - l0) * args.steps // (args.steps + args.warmup)
        ms_kernel = ms
        owned = N

        # ---- fp32 vmult ----
        x32 = x.float()
        y32 = torch.empty_like(x32)
        ms32, _ = timed(lambda: ctx.apply_stokes(level, x32, out=y32), args.steps)
        extra["fp32_vmult"] = {"value": N / (ms32 * 1e-3), "unit": "DoF/s", "ms": ms32}

        # ---- fp32 smoothing step (8 colours: residual + patch solve each) ----
        b32 = ctx.apply_stokes(level, x32)
        xs = torch.zeros_like(b32)
        sm_steps = max(3, min(args.steps, 20))
        ctx.smoother_stats(reset=True)
        ms_smooth, _ = timed(lambda: ctx.smooth(level, xs, b32, zero_init=True), sm_steps)
        npatch, cgit = ctx.smoother_stats(reset=True)
        fl = smoother_flops(k, npatch, cgit) / (sm_steps + args.warmup)
        sm_tf = fl / (ms_smooth * 1e-3) / 1e12
        extra["smoother_fp32"] = {"value": N / (ms_smooth * 1e-3), "unit": "DoF/s", "ms_per_step": ms_smooth,
                                  "ns_per_dof": ms_smooth * 1e6 / N, "timed_steps": sm_steps,
                                  "mean_inner_cg_iterations": cgit / max(npatch, 1), "cg_tol": 1e-5,
                                  "roofline": {"bound": "fp32 fma", "achieved_tflops": sm_tf,
                                               "peak_tflops": FP32_PEAK_TFLOPS, "frac": sm_tf / FP32_PEAK_TFLOPS,
                                               "algorithmic_flops_per_step": fl,
                                               "note": "whole step incl. the 8 residual launches; patch-kernel "
                                                       "flops only (bench.smoother_flops)"}}

        # the smoothing step with the loose inner tolerance the tuned solve uses (FGMRES iterations unchanged)
        ctx_l = smg.Context(k, level, device=local, cg_max_iter=30, cg_tol=1e-2, cg_fixed=False, cg_precond=1)
        ctx_l.smoother_stats(reset=True)
        ms_sl, _ = timed(lambda: ctx_l.smooth(level, xs, b32, zero_init=True), sm_steps)
        npl, cgl = ctx_l.smoother_stats(reset=True)
        extra["smoother_fp32_inner_cg_tol_1e-2"] = {"value": N / (ms_sl * 1e-3), "unit": "DoF/s", "ms_per_step": ms_sl,
                                                    "mean_inner_cg_iterations": cgl / max(npl, 1)}
        del ctx_l

        # ---- intergrid transfer (fp32, level 5 <-> 4): restrict r_c = P^T r_f, prolongate x_f += P x_c ----
        rc32 = torch.zeros(ctx.sizes(level - 1)[4], dtype=torch.float32, device="cuda")
        ms_r, _ = timed(lambda: ctx.restrict(level - 1, b32, out=rc32), args.steps)
        ms_p, _ = timed(lambda: ctx.prolongate_add(level - 1, xs, rc32), args.steps)
        peak_gbs, _ = measured_peaks()
        nc = ctx.sizes(level - 1)[4]
        br, bp = 4 * (N + nc), 4 * (2 * N + nc)  # algorithmic bytes: read fine + write coarse; RMW fine + read coarse
        extra["transfer_fp32"] = {
            "restrict": {"ms": ms_r, "gbs": br / ms_r / 1e6, "hbm_frac": br / ms_r / 1e6 / peak_gbs,
                         "algorithmic_bytes": br},
            "prolongate_add": {"ms": ms_p, "gbs": bp / ms_p / 1e6, "hbm_frac": bp / ms_p / 1e6 / peak_gbs,
                               "algorithmic_bytes": bp}}

        # ---- MG-FGMRES solve (mixed precision: fp64 Krylov, fp32 V-cycle) ----
        if not args.no_solve:
            b = ctx.apply_stokes(level, x)
            ctx.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            xsol, it, hist = ctx.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)
            torch.cuda.synchronize()
            ts = time.perf_counter() - t0
            nu = -8.0 / np.log10((hist[-1] / hist[0]) ** (1.0 / it)) if it > 0 and hist[-1] > 0 else None
            extra["solve"] = {"iterations": it, "rel_residual": float(hist[-1] / hist[0]), "fractional_count_nu": nu,
                              "time_s": ts, "ns_per_dof": ts / N * 1e9, "tol": 1e-8, "inner_cg_tol": 1e-5,
                              "precision": "fp64 FGMRES + fp32 V-cycle"}
            # the same solve with a loose inner patch-CG tolerance: FGMRES is flexible, the outer iteration
            # count stays (profiles/r02/cgtol_sweep.txt) while the smoothing work drops
            ctx2 = smg.Context(k, level, device=local, cg_max_iter=30, cg_tol=1e-2, cg_fixed=False, cg_precond=1)
            ctx2.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, it2, hist2 = ctx2.solve(level, b, 1e-8, 30, smg.F32, allow_not_converged=True)
            torch.cuda.synchronize()
            ts2 = time.perf_counter() - t0
            extra["solve_inner_cg_tol_1e-2"] = {"iterations": it2, "rel_residual": float(hist2[-1] / hist2[0]),
                                                "time_s": ts2, "ns_per_dof": ts2 / N * 1e9, "tol": 1e-8,
                                                "inner_cg_tol": 1e-2}
            del ctx2

        # ---- e2e: host BlockVector buffers through the C ABI, copies inside the timed region ----
        s = ctx.sizes(level)
        xbn = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
        ybn = [torch.empty(s[i], dtype=torch.float64, pin_memory=True).numpy() for i in range(4)]
        for i, blk in enumerate(smg.to_blockvector(x.cpu().numpy(), k, level)):
            xbn[i][:] = blk
        for _ in range(args.warmup):
            ctx.vmult_host(level, xbn, smg.F64, out=ybn)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ctx.vmult_host(level, xbn, smg.F64, out=ybn)
        te = (time.perf_counter() - t0) / args.steps
        e2e = {"value": N / te, "unit": "DoF/s", "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
               "path": "smg_vmult_host: BlockVector host arrays (pinned), pipelined over z-chunks: H2D / vmult / D2H on three streams"}
        parallelism = "single GPU"
    else:
        # ---- z-slab partition of the same global problem through the C ABI's multi-GPU driver
        #      (csrc/dist.cu: NCCL ghost exchange + slab operator, slab V-cycle and FGMRES in C++) ----
        from paper_2410_09497_b200 import dist as sd
        D = sd.DistContext(ctx, world, rank)
        transport = "library NCCL"
        if args.dist_backend == "nccl":
            try:
                D.init_nccl()
            except Exception as e:  # noqa: BLE001 -- keep the run alive on the torch.distributed NCCL transport
                print(f"[rank {rank}] in-library NCCL unavailable ({e}); torch.distributed NCCL transport",
                      file=sys.stderr)
                D = sd.DistContext(ctx, world, rank).init_torch_transport()
                transport = "torch.distributed NCCL callbacks"
        else:
            D.init_torch_transport()  # gloo: host-staged callbacks (multi-rank logic runs on one GPU)
            transport = "gloo callbacks (host-staged)"
        extra["dist_transport"] = transport
        (z0, z1, zlo, zhi), hs = D.held(level)
        xsl = D.extract(level, x)
        # correctness of the partitioned operator against the whole-level operator on the owned rows
        yref = ctx.apply_stokes(level, x)
        ysl = torch.zeros_like(xsl)
        D.vmult(level, ysl, xsl)
        yfull = torch.zeros_like(yref)
        D.insert_owned(level, yfull, ysl)
        mask = torch.zeros_like(yref)
        D.insert_owned(level, mask, torch.ones_like(ysl))
        err = float(((yfull - yref) * mask).abs().max()) / max(float(yref.abs().max()), 1e-300)
        extra["slab_check_rel_err"] = max_over_ranks(err)
        del yfull, mask
        if not args.no_solve:
            bh = D.extract(level, yref)
            D.solve(bh, 1e-8, 30, smg.F32)  # warm-up
            barrier()
            t0 = time.perf_counter()
            _, it, hist = D.solve(bh, 1e-8, 30, smg.F32)
            torch.cuda.synchronize()
            ts = max_over_ranks(time.perf_counter() - t0)
            extra["solve"] = {"iterations": it, "rel_residual": float(hist[-1] / hist[0]), "time_s": ts,
                              "ns_per_dof": ts / N * 1e9, "tol": 1e-8,
                              "precision": "fp64 FGMRES + fp32 V-cycle, z-slab multigrid in C++ (smg_dist_solve)"}
        del yref, x
        torch.cuda.empty_cache()
        l0 = ctx.launch_count
        ms, clk = timed(lambda: D.vmult(level, ysl, xsl), args.steps, clocks=True)
        launches = (ctx.launch_count - l0) * args.steps // (args.steps + args.warmup)
        # kernel-only: the slab operator without the exchange (smg_residual_held on the owned rows)
        from paper_2410_09497_b200 import lib, _ptr
        ms_kernel, _ = timed(lambda: lib().smg_residual_held(ctx._h, level, smg.F64, _ptr(ysl), None, _ptr(xsl), zlo,
                                                             zhi, z0, z1), args.steps)
        H = k + 1
        n_ = (2 << level) * H
        owned = sum((z1 - z0) * H * p for p in ((n_ + 1) * n_, n_ * (n_ + 1), n_ * n_, n_ * n_))
        xh = torch.empty(xsl.numel(), dtype=torch.float64, pin_memory=True)
        yh = torch.empty(xsl.numel(), dtype=torch.float64, pin_memory=True)
        xh.copy_(xsl)

        def e2e_step():
            xsl.copy_(xh, non_blocking=True)
            D.vmult(level, ysl, xsl)
            yh.copy_(ysl, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        for _ in range(args.warmup):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        te = max_over_ranks((time.perf_counter() - t0) / args.steps)
        e2e = {"value": N / te, "unit": "DoF/s", "h2d_bytes_per_step": 8 * xsl.numel(),
               "d2h_bytes_per_step": 8 * xsl.numel(),
               "path": "per rank: pinned held slab -> H2D -> smg_dist_vmult (NCCL ghost exchange + slab operator) -> D2H"}
        extra["kernel_ms"] = ms_kernel
        extra["slab"] = {"z_cells": [z0, z1], "held_cells": [zlo, zhi], "owned_dofs": owned, "held_dofs": hs[4]}
        parallelism = f"z-slabs x{world} (C-ABI dist driver, NCCL ghost exchange)"
    value = N / (ms * 1e-3)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_src = measured_peaks()
    bytes_per_launch = 16 * owned  # algorithmic: read x + write y of the owned DoF, fp64
    achieved = bytes_per_launch / (ms_kernel * 1e-3) / 1e9
    traffic = ncu_traffic(f"k{k}_l{level}_f64") if world == 1 else None
    cpu = None if (args.no_cpu or world > 1) else cpu_baseline(k, level)
    out = {
        "metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (uniform random x, seed 1234)",
        "config": dict(workload_config(k, level), parallelism=parallelism),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "kernel": f"stokes_vmult_kernel<double,{k}> ({SHAPES.get(k, 'see DESIGN.md')})"},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches,
    }
    # compute side of the roofline: algorithmic flops of the Kronecker-form operator (SURVEY.md §8(d):
    # 19.5 k + 33 per DoF) against the FP64 FMA peak measured with tools/fma_peak.cu
    flops = (19.5 * k + 33) * owned
    tflops = flops / (ms_kernel * 1e-3) / 1e12
    out["roofline"]["compute"] = {"algorithmic_flops_per_launch": flops, "achieved_tflops": tflops,
                                  "fp64_peak_tflops": FP64_PEAK_TFLOPS, "frac": tflops / FP64_PEAK_TFLOPS,
                                  "peak_source": "measured, profiles/r01/fma_peaks.txt (tools/fma_peak.cu)"}
    out.update(extra)
    print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
