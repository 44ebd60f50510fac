"""Multigrid and MG-preconditioned FGMRES on z-slabs.

Every level l above the agglomeration level is split like the finest one (owned cells
[z0 >> (L-l), z1 >> (L-l))); MG vectors hold GHOST = 3 cell layers beyond each interior end:
  * smoothing, per colour: ghost exchange of x, residual on the rows of cells [z0-2, z1+1), then the
    patches with vertex planes z0..z1 (the two face patches are computed identically by both
    neighbours, so no update is sent back; SPEC.md:424 frozen residual per colour);
  * restriction reads fine cells 2c0-2 .. 2c1 (hence the residual on [z0-2, z1+1) and GHOST = 3);
  * prolongation adds into the owned fine rows only; the next smoothing exchanges first;
  * at the agglomeration level (slabs thinner than 4 cells or not nested) the level's right-hand side
    is summed over the ranks into a full vector and the rest of the V-cycle runs replicated with the
    single-GPU path (the coarse levels are tiny).
A SlabMG drives either ONE part per process (torch.distributed P2P / all-reduce between ranks, NCCL on
GPUs) or, for tests on one device, ALL parts of a virtual partition in one process (exchanges become
device copies). FGMRES (fgmres) follows smg_solve: right preconditioning, MGS + one re-orthogonalisation,
fp64 Krylov vectors, V-cycle in fp32 or fp64, dots all-reduced over the owned rows.
"""
import ctypes
import math

import numpy as np

from . import F32, F64, SMG_OK, NotConverged, _ptr, lib, pressure_node_weights
from .slab import partition

GHOST = 3


class LevelSlab:
    """one part's cells of one level: owned [z0, z1), held [zlo, zhi) (layout of smg_held_sizes)."""

    def __init__(self, k, level, z0, z1, ghost=GHOST):
        self.k, self.level, self.H = k, level, k + 1
        self.m = 2 << level
        self.n = self.m * self.H
        self.z0, self.z1 = z0, z1
        self.zlo, self.zhi = max(z0 - ghost, 0), min(z1 + ghost, self.m)
        n, nz = self.n, (self.zhi - self.zlo) * self.H
        self.plane = [(n + 1) * n, n * (n + 1), n * n, n * n]
        self.planes = [nz, nz, nz + 1, nz]
        self.size = [p * q for p, q in zip(self.plane, self.planes)]
        self.off = list(np.cumsum([0] + self.size[:3]))
        self.total = int(sum(self.size))

    def block(self, v, c):
        return v[self.off[c]:self.off[c] + self.size[c]].view(self.planes[c], self.plane[c])

    def cells(self, a, b):
        """local plane range of the held cells [a, b)."""
        return (a - self.zlo) * self.H, (b - self.zlo) * self.H

    def owned_planes(self, c):
        a, b = self.cells(self.z0, self.z1)
        return a, b + (1 if c == 2 and self.z1 == self.m else 0)

    def extract(self, g):
        """held part of a full-level vector (torch)."""
        import torch
        full = LevelSlab(self.k, self.level, 0, self.m, 0)
        parts = []
        for c in range(4):
            lo = self.zlo * self.H
            parts.append(full.block(g, c)[lo:lo + self.planes[c]].reshape(-1))
        return torch.cat(parts)

    def add_owned_into(self, g, v):
        full = LevelSlab(self.k, self.level, 0, self.m, 0)
        for c in range(4):
            a, b = self.owned_planes(c)
            lo = self.zlo * self.H
            full.block(g, c)[lo + a:lo + b] += self.block(v, c)[a:b]


class SlabMG:
    def __init__(self, ctx, level, bounds, parts, group=None, world=None):
        """bounds: owned finest-level cells of every rank; parts: the ranks handled by this process
        (one rank per process under torch.distributed, or all of them for a virtual partition)."""
        self.ctx, self.L, self.k = ctx, level, ctx.degree
        self.bounds, self.parts, self.group = bounds, list(parts), group
        self.world = world or len(bounds)
        self.virtual = len(self.parts) > 1
        if self.virtual and len(self.parts) != self.world:
            raise ValueError("a virtual partition must hold every part")
        # finest levels that stay partitioned: every slab nests (z0, z1 divisible) and has >= 4 cells
        self.la = level
        for l in range(level, 0, -1):
            s = 1 << (level - l)
            if all(z0 % s == 0 and z1 % s == 0 and (z1 - z0) // s >= 4 for z0, z1 in bounds):
                self.la = l - 1
            else:
                break
        if self.la >= level:
            raise ValueError("the finest level is too thin to partition (>= 4 cells per slab needed)")
        self.slabs = {p: {l: LevelSlab(self.k, l, bounds[p][0] >> (level - l), bounds[p][1] >> (level - l))
                          for l in range(self.la + 1, level + 1)} for p in self.parts}
        self._vec = {}

    # ---- buffers ----
    def vec(self, p, l, dtype, name):
        import torch
        key = (p, l, dtype, name)
        if key not in self._vec:
            self._vec[key] = torch.zeros(self.slabs[p][l].total, dtype=dtype, device=f"cuda:{self.ctx.device}")
        return self._vec[key]

    def new(self, l, dtype):
        import torch
        return {p: torch.zeros(self.slabs[p][l].total, dtype=dtype, device=f"cuda:{self.ctx.device}")
                for p in self.parts}

    # ---- communication ----
    def exchange(self, l, vs):
        """refresh GHOST cell layers of the part vectors vs[p] from the neighbours' owned cells."""
        self.exchange_finish(self.exchange_start(l, vs))

    @staticmethod
    def exchange_finish(works):
        for w in works or []:
            w.wait()  # the current stream waits for the NCCL transfers

    def exchange_start(self, l, vs):
        """post the ghost exchange; returns NCCL work handles to finish later (None: already done)."""
        if self.virtual:
            for p in self.parts:
                S = self.slabs[p][l]
                for q in (p - 1, p + 1):
                    if q < 0 or q >= self.world:
                        continue
                    T = self.slabs[q][l]
                    a, b = max(S.zlo, T.z0), min(S.zhi, T.z1)  # my ghost cells owned by q
                    if a >= b:
                        continue
                    for c in range(4):
                        sa, sb = S.cells(a, b)
                        ta, tb = T.cells(a, b)
                        S.block(vs[p], c)[sa:sb] = T.block(vs[q], c)[ta:tb]
            return None
        import torch.distributed as dist
        if dist.get_backend(self.group) == "gloo" and any(v.is_cuda for v in vs.values()):
            # gloo has no CUDA P2P: stage through host memory (logic checks on single-GPU boxes)
            hs = {p: v.cpu() for p, v in vs.items()}
            self.exchange(l, hs)
            for p in vs:
                vs[p].copy_(hs[p])
            return None
        ops = []
        for p in self.parts:
            S = self.slabs[p][l]
            v = vs[p]
            for q in (p - 1, p + 1):
                if q < 0 or q >= self.world:
                    continue
                z0q, z1q = self.bounds[q][0] >> (self.L - l), self.bounds[q][1] >> (self.L - l)
                # send my owned cells inside q's held range; receive q's owned cells inside mine
                sa, sb = max(S.z0, max(z0q - GHOST, 0)), min(S.z1, min(z1q + GHOST, S.m))
                ra, rb = max(S.zlo, z0q), min(S.zhi, z1q)
                for c in range(4):
                    if sa < sb:
                        a, b = S.cells(sa, sb)
                        ops.append(dist.P2POp(dist.isend, S.block(v, c)[a:b], q, self.group))
                    if ra < rb:
                        a, b = S.cells(ra, rb)
                        ops.append(dist.P2POp(dist.irecv, S.block(v, c)[a:b], q, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def allreduce_full(self, l, contrib):
        """sum over ranks of full-level vectors (agglomeration)."""
        if self.virtual:
            return contrib
        import torch.distributed as dist
        if dist.get_backend(self.group) == "gloo" and contrib.is_cuda:
            h = contrib.cpu()
            dist.all_reduce(h, group=self.group)
            contrib.copy_(h)
            return contrib
        dist.all_reduce(contrib, group=self.group)
        return contrib

    def dot(self, l, a, b):
        out, tot = ctypes.c_double(), 0.0
        for p in self.parts:
            S = self.slabs[p][l]
            prec = self.ctx._prec(a[p])
            self.ctx._sync_stream()
            self.ctx._check(lib().smg_dot_held(self.ctx._h, l, prec, _ptr(a[p]), _ptr(b[p]), S.zlo, S.zhi, S.z0, S.z1,
                                               ctypes.byref(out)))
            tot += out.value
        if not self.virtual and self.world > 1:
            import torch
            import torch.distributed as dist
            gloo = dist.get_backend(self.group) == "gloo"
            t = torch.tensor([tot], dtype=torch.float64, device="cpu" if gloo else f"cuda:{self.ctx.device}")
            dist.all_reduce(t, group=self.group)
            tot = float(t.item())
        return tot

    # ---- operators ----
    def residual(self, l, r, b, x, c0, c1, skip=None):
        """r = b - A x on the rows of cells [z0 + c0, z1 + c1) (clipped to the level); skip = (s0, s1)
        leaves out the rows [z0 + s0, z1 + s1) (computed earlier)."""
        for p in self.parts:
            S = self.slabs[p][l]
            a0, a1 = max(S.z0 + c0, 0), min(S.z1 + c1, S.m)
            spans = [(a0, a1)]
            if skip is not None:
                s0, s1 = max(S.z0 + skip[0], a0), min(S.z1 + skip[1], a1)
                if s0 < s1:
                    spans = [(a0, s0), (s1, a1)]
            for u0, u1 in spans:
                if u0 < u1:
                    self.ctx._check(lib().smg_residual_held(self.ctx._h, l, self.ctx._prec(x[p]), _ptr(r[p]),
                                                            _ptr(b[p]), _ptr(x[p]), S.zlo, S.zhi, u0, u1))

    def vmult(self, l, y, x):
        """y = A x on the owned rows (x ghosts must be current)."""
        for p in self.parts:
            S = self.slabs[p][l]
            self.ctx._check(lib().smg_residual_held(self.ctx._h, l, self.ctx._prec(x[p]), _ptr(y[p]), None,
                                                    _ptr(x[p]), S.zlo, S.zhi, S.z0, S.z1))

    def smooth(self, l, x, b, r):
        for col in range(8):
            # the residual rows that need no ghost cell are computed while the exchange runs
            works = self.exchange_start(l, x)
            self.residual(l, r, b, x, 1, -1)
            self.exchange_finish(works)
            self.residual(l, r, b, x, -2, 1, skip=(1, -1))
            for p in self.parts:
                S = self.slabs[p][l]
                self.ctx._check(lib().smg_smooth_colour_held(self.ctx._h, l, self.ctx._prec(x[p]), col, _ptr(x[p]),
                                                             _ptr(r[p]), S.zlo, S.zhi, S.z0, S.z1))

    def vcycle(self, l, b, dtype):
        """x = V(b); b holds valid owned rows (ghosts are refreshed here)."""
        import torch
        if l == self.la:
            full = torch.zeros(self.ctx.sizes(l)[4], dtype=dtype, device=f"cuda:{self.ctx.device}")
            for p in self.parts:
                S = LevelSlab(self.k, l, self.bounds[p][0] >> (self.L - l), self.bounds[p][1] >> (self.L - l))
                S.add_owned_into(full, b[p])
            full = self.allreduce_full(l, full)
            xf = self.ctx.vcycle(l, full)
            return {p: LevelSlab(self.k, l, self.bounds[p][0] >> (self.L - l),
                                 self.bounds[p][1] >> (self.L - l)).extract(xf) for p in self.parts}
        x = {p: self.vec(p, l, dtype, "x").zero_() for p in self.parts}
        r = {p: self.vec(p, l, dtype, "r") for p in self.parts}
        self.exchange(l, b)
        self.smooth(l, x, b, r)
        self.exchange(l, x)
        self.residual(l, r, b, x, -2, 1)
        lc = l - 1
        if lc == self.la:
            bc = {}
            for p in self.parts:
                Sc = LevelSlab(self.k, lc, self.bounds[p][0] >> (self.L - lc), self.bounds[p][1] >> (self.L - lc))
                bc[p] = torch.zeros(Sc.total, dtype=dtype, device=b[p].device)
                S = self.slabs[p][l]
                self.ctx._check(lib().smg_restrict_held(self.ctx._h, lc, self.ctx._prec(r[p]), _ptr(bc[p]), _ptr(r[p]),
                                                        S.zlo, S.zhi, Sc.zlo, Sc.zhi, Sc.z0, Sc.z1))
        else:
            bc = {p: self.vec(p, lc, dtype, "b") for p in self.parts}
            for p in self.parts:
                S, Sc = self.slabs[p][l], self.slabs[p][lc]
                self.ctx._check(lib().smg_restrict_held(self.ctx._h, lc, self.ctx._prec(r[p]), _ptr(bc[p]), _ptr(r[p]),
                                                        S.zlo, S.zhi, Sc.zlo, Sc.zhi, Sc.z0, Sc.z1))
        xc = self.vcycle(lc, bc, dtype)
        for p in self.parts:
            S = self.slabs[p][l]
            Sc = self.slabs[p][lc] if lc > self.la else LevelSlab(self.k, lc, self.bounds[p][0] >> (self.L - lc),
                                                                   self.bounds[p][1] >> (self.L - lc))
            self.ctx._check(lib().smg_prolongate_add_held(self.ctx._h, lc, self.ctx._prec(x[p]), _ptr(x[p]), _ptr(xc[p]),
                                                          S.zlo, S.zhi, Sc.zlo, Sc.zhi, S.z0, S.z1))
        self.smooth(l, x, b, r)
        return {p: x[p].clone() for p in self.parts}

    def allreduce_scalar(self, v):
        if self.virtual or self.world == 1:
            return v
        import torch
        import torch.distributed as dist
        gloo = dist.get_backend(self.group) == "gloo"
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if gloo else f"cuda:{self.ctx.device}")
        dist.all_reduce(t, group=self.group)
        return float(t.item())

    def project_zero_mean(self, x):
        """Subtract the mass-weighted pressure mean (project_zero_mean SPEC.md:212-220) from every held
        pressure row; the weighted sum runs over the owned rows and is all-reduced, so all ranks subtract
        the same constant -- the one smg_solve subtracts on one GPU."""
        import torch
        L, H = self.L, self.k + 1
        w1 = pressure_node_weights(self.k)
        tot = 0.0
        for p in self.parts:
            S = self.slabs[p][L]
            a, b = S.owned_planes(3)
            pb = S.block(x[p], 3)[a:b]
            dev = pb.device
            wz = torch.tensor(w1[(np.arange(S.zlo * H + a, S.zlo * H + b)) % H], dtype=torch.float64, device=dev)
            wn = torch.tensor(w1[np.arange(S.n) % H], dtype=torch.float64, device=dev)
            wxy = torch.outer(wn, wn).reshape(-1)
            tot += float((wz[:, None] * wxy[None, :] * pb.double()).sum())
        tot = self.allreduce_scalar(tot)
        mean = tot / (float(w1.sum()) ** 3 * float(2 << L) ** 3)
        for p in self.parts:
            self.slabs[p][L].block(x[p], 3).sub_(mean)
        return x

    # ---- FGMRES (smg_solve semantics) ----
    def solve(self, b, tol=1e-8, max_iter=50, vcycle_precision=F32, allow_not_converged=False):
        """b: {part: fp64 held vector with valid owned rows}. Returns ({part: x}, iterations, history).
        As smg_solve: the mass-weighted pressure mean of x is removed, and NotConverged is raised if the
        relative residual did not reach `tol` within max_iter (unless allow_not_converged)."""
        import torch
        L = self.L
        d32 = torch.float32 if vcycle_precision == F32 else torch.float64
        beta = math.sqrt(self.dot(L, b, b))
        hist = [beta]
        x = {p: torch.zeros_like(b[p]) for p in self.parts}
        if beta == 0.0:
            return x, 0, hist
        V = [{p: b[p] / beta for p in self.parts}]
        Z = []
        Hm = np.zeros((max_iter + 1, max_iter))
        cs, sn, g = np.zeros(max_iter), np.zeros(max_iter), np.zeros(max_iter + 1)
        g[0] = beta
        it = 0
        converged = False
        for j in range(max_iter):
            z = self.vcycle(L, {p: V[j][p].to(d32) for p in self.parts}, d32)
            Z.append({p: z[p].double() for p in self.parts})
            w = {p: torch.zeros_like(b[p]) for p in self.parts}
            self.exchange(L, Z[j])
            self.vmult(L, w, Z[j])
            for _ in range(2):
                for i in range(j + 1):
                    hij = self.dot(L, w, V[i])
                    Hm[i, j] += hij
                    for p in self.parts:
                        w[p] -= hij * V[i][p]
            wn = math.sqrt(self.dot(L, w, w))
            Hm[j + 1, j] = wn
            for i in range(j):
                t = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -sn[i] * Hm[i, j] + cs[i] * Hm[i + 1, j]
                Hm[i, j] = t
            den = math.hypot(Hm[j, j], Hm[j + 1, j])
            cs[j], sn[j] = Hm[j, j] / den, Hm[j + 1, j] / den
            Hm[j, j], Hm[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it = j + 1
            hist.append(abs(g[j + 1]))
            if abs(g[j + 1]) <= tol * beta or wn == 0.0:
                converged = True
                break
            V.append({p: w[p] / wn for p in self.parts})
        y = np.zeros(it)
        for i in range(it - 1, -1, -1):
            y[i] = (g[i] - Hm[i, i + 1:it] @ y[i + 1:it]) / Hm[i, i]
        for i in range(it):
            for p in self.parts:
                x[p] += y[i] * Z[i][p]
        self.project_zero_mean(x)
        if not converged and not allow_not_converged:
            raise NotConverged(-101, f"slab FGMRES: relative residual {hist[-1] / beta:.3e} > {tol:g} "
                                     f"after {it} iterations")
        return x, it, hist


def virtual_partition(ctx, level, nparts):
    """SlabMG over nparts virtual ranks of one device (tests)."""
    bounds = partition(level, nparts)
    return SlabMG(ctx, level, bounds, range(nparts))
