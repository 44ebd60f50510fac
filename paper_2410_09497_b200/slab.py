"""z-slab partition of a level across ranks (one GPU per rank) with ghost-layer exchange.

SURVEY.md §8(e) / DESIGN.md §6: the cells of the unit cube are split into contiguous z-slabs; a slab
vector holds the owned cells [z0, z1) plus one ghost cell layer on each interior side, in the layout
of include/smg_b200.h (smg_slab_sizes): each block [u_x, u_y, u_z, p] keeps its global x/y extents and
the z node planes of the held cells (u_z: one extra top plane). Before each operator apply the ghost
layers are refreshed from the neighbours (one cell layer = k+1 node planes per block, contiguous
in memory, so every message is a plain slice: no packing). The exchange runs over torch.distributed
(NCCL between GPUs over NVLink; gloo on CPU for the host-logic tests).
"""
import ctypes

import numpy as np

from . import F32, F64, SMG_OK, _ptr, level_sizes, lib


def partition(level, world, multiple=4):
    """Owned cell ranges [z0, z1) per rank: contiguous, as even as possible, every interior boundary
    on a multiple of `multiple` cells (the vmult kernel's largest brick depth), so slab bricks tile
    exactly. Raises ValueError if the level has too few cells for `world` slabs."""
    m = 2 << level
    units = m // multiple if m % multiple == 0 else 0
    if units < world:
        if m >= world and multiple > 1:
            return partition(level, world, multiple // 2)
        raise ValueError(f"level {level} ({m} cells) cannot be split into {world} slabs")
    base, extra = divmod(units, world)
    bounds, z = [], 0
    for r in range(world):
        z1 = z + (base + (1 if r < extra else 0)) * multiple
        bounds.append((z, z1))
        z = z1
    return bounds


class SlabLayout:
    """Python mirror of the slab LevelLayout (csrc/smg_internal.cuh)."""

    def __init__(self, degree, level, z0, z1):
        self.k, self.level = degree, level
        self.H = degree + 1
        self.m = 2 << level
        self.n = self.m * self.H
        self.z0, self.z1 = z0, z1
        self.zlo, self.zhi = max(z0 - 1, 0), min(z1 + 1, self.m)
        n, H = self.n, self.H
        nz = (self.zhi - self.zlo) * H
        self.plane = [(n + 1) * n, n * (n + 1), n * n, n * n]
        self.planes = [nz, nz, nz + 1, nz]
        self.size = [p * q for p, q in zip(self.plane, self.planes)]
        self.off = list(np.cumsum([0] + self.size[:3]))
        self.total = int(sum(self.size))

    def block(self, v, c):
        """block c of a flat slab vector as a (planes, plane) view."""
        return v[self.off[c]:self.off[c] + self.size[c]].reshape(self.planes[c], self.plane[c])

    def cell_planes(self, z):
        """local plane range [a, b) of global cell z (k+1 planes)."""
        a = (z - self.zlo) * self.H
        return a, a + self.H

    def owned_planes(self, c):
        a, _ = self.cell_planes(self.z0)
        b = (self.z1 - self.zlo) * self.H + (1 if c == 2 and self.z1 == self.m else 0)
        return a, b

    # ---- global <-> slab (tests, set-up and gather of results) ----
    def extract(self, g):
        """slab vector (owned + ghost cells) cut from a flat GLOBAL level vector (numpy or torch)."""
        glob = SlabLayout(self.k, self.level, 0, self.m)
        parts = []
        for c in range(4):
            gb = glob.block(g, c)
            lo = self.zlo * self.H
            parts.append(gb[lo:lo + self.planes[c]].reshape(-1))
        if isinstance(g, np.ndarray):
            return np.concatenate(parts)
        import torch
        return torch.cat(parts)

    def insert_owned(self, g, v):
        """write the owned rows of slab vector v into the flat GLOBAL vector g."""
        glob = SlabLayout(self.k, self.level, 0, self.m)
        for c in range(4):
            a, b = self.owned_planes(c)
            lo = self.zlo * self.H
            glob.block(g, c)[lo + a:lo + b] = self.block(v, c)[a:b]
        return g


class HaloExchange:
    """Ghost-layer exchange of slab vectors between neighbouring ranks (torch.distributed P2P)."""

    def __init__(self, layout, rank, world, group=None):
        self.lay, self.rank, self.world, self.group = layout, rank, world, group

    def _ops(self, v):
        import torch.distributed as dist
        L, ops = self.lay, []
        for c in range(4):
            blk = L.block(v, c)
            if self.rank > 0:  # my first owned cell -> rank-1 ; rank-1's last owned cell -> my ghost below
                a, b = L.cell_planes(L.z0)
                ops.append(dist.P2POp(dist.isend, blk[a:b], self.rank - 1, self.group))
                a, b = L.cell_planes(L.zlo)
                ops.append(dist.P2POp(dist.irecv, blk[a:b], self.rank - 1, self.group))
            if self.rank < self.world - 1:
                a, b = L.cell_planes(L.z1 - 1)
                ops.append(dist.P2POp(dist.isend, blk[a:b], self.rank + 1, self.group))
                a, b = L.cell_planes(L.zhi - 1)
                ops.append(dist.P2POp(dist.irecv, blk[a:b], self.rank + 1, self.group))
        return ops

    def exchange(self, v):
        import torch.distributed as dist
        if v.is_cuda and dist.get_backend(self.group) == "gloo":
            # gloo has no CUDA P2P: stage through host memory (test mode on single-GPU boxes)
            h = v.cpu()
            self.exchange(h)
            v.copy_(h)
            return v
        ops = self._ops(v)
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return v

    def start(self, v):
        """post the exchange and return its work handles (NCCL runs it on its own stream); None when the
        backend cannot overlap (gloo: done synchronously here)."""
        import torch.distributed as dist
        if dist.get_backend(self.group) == "gloo":
            self.exchange(v)
            return None
        ops = self._ops(v)
        return dist.batch_isend_irecv(ops) if ops else []

    @staticmethod
    def finish(works):
        for w in works or []:
            w.wait()  # the current stream waits for the exchange


def exchange_local(layouts, vecs):
    """single-process ghost exchange between slab vectors of one device (tests, virtual slabs)."""
    for r in range(len(layouts) - 1):
        lo, hi = layouts[r], layouts[r + 1]
        for c in range(4):
            a, b = lo.cell_planes(lo.z1 - 1)   # my last owned cell
            a2, b2 = hi.cell_planes(hi.zlo)     # the upper neighbour's ghost below
            hi.block(vecs[r + 1], c)[a2:b2] = lo.block(vecs[r], c)[a:b]
            a, b = hi.cell_planes(hi.z0)        # the upper neighbour's first owned cell
            a2, b2 = lo.cell_planes(lo.zhi - 1)  # my ghost above
            lo.block(vecs[r], c)[a2:b2] = hi.block(vecs[r + 1], c)[a:b]
    return vecs


def slab_sizes(degree, level, z0, z1):
    s = (ctypes.c_int64 * 5)()
    if lib().smg_slab_sizes(degree, level, z0, z1, s) != SMG_OK:
        raise ValueError("invalid slab")
    return [int(v) for v in s]


class SlabOperator:
    """The Stokes operator of one rank's slab: exchange ghosts, apply, owned-row dots (all-reduced)."""

    def __init__(self, ctx, level, z0, z1, rank=0, world=1, group=None):
        self.ctx, self.level = ctx, level
        self.lay = SlabLayout(ctx.degree, level, z0, z1)
        if slab_sizes(ctx.degree, level, z0, z1)[4] != self.lay.total:
            raise RuntimeError("slab layout mismatch between the library and slab.py")
        self.halo = HaloExchange(self.lay, rank, world, group) if world > 1 else None
        self.world = world

    def new_vector(self, dtype=None):
        import torch
        return torch.zeros(self.lay.total, dtype=dtype or torch.float64, device=f"cuda:{self.ctx.device}")

    def exchange(self, x):
        if self.halo is not None:
            self.halo.exchange(x)
        return x

    def _rows(self, y, x, c0, c1, b=None):
        L = self.lay
        if c0 >= c1:
            return
        self.ctx._check(lib().smg_residual_held(self.ctx._h, self.level, self.ctx._prec(x), _ptr(y),
                                                None if b is None else _ptr(b), _ptr(x), L.zlo, L.zhi, c0, c1))

    def vmult(self, y, x, exchange=True, overlap=True):
        """y = A x on the owned rows. With an exchange, the rows that do not touch a ghost cell are
        computed while NCCL moves the ghost layers (interior first, then the two boundary cell layers)."""
        p = self.ctx._prec(x)
        self.ctx._sync_stream()
        L = self.lay
        if not exchange or self.halo is None or not overlap or L.z1 - L.z0 < 3:
            if exchange:
                self.exchange(x)
            self.ctx._check(lib().smg_vmult_slab(self.ctx._h, self.level, p, _ptr(y), _ptr(x), L.z0, L.z1))
            return y
        works = self.halo.start(x)
        lo = L.z0 + (1 if L.zlo < L.z0 else 0)   # first cell whose rows need no ghost below
        hi = L.z1 - (1 if L.zhi > L.z1 else 0)   # one past the last cell needing no ghost above
        self._rows(y, x, lo, hi)
        self.halo.finish(works)
        self._rows(y, x, L.z0, lo)
        self._rows(y, x, hi, L.z1)
        return y

    def residual(self, r, b, x, exchange=True):
        if exchange:
            self.exchange(x)
        p = self.ctx._prec(x)
        self.ctx._sync_stream()
        self.ctx._check(lib().smg_residual_slab(self.ctx._h, self.level, p, _ptr(r), _ptr(b), _ptr(x),
                                                self.lay.z0, self.lay.z1))
        return r

    def dot(self, a, b):
        out = ctypes.c_double()
        self.ctx._sync_stream()
        self.ctx._check(lib().smg_dot_slab(self.ctx._h, self.level, self.ctx._prec(a), _ptr(a), _ptr(b),
                                           self.lay.z0, self.lay.z1, ctypes.byref(out)))
        if self.world > 1:
            import torch
            import torch.distributed as dist
            gloo = dist.get_backend(self.halo.group) == "gloo"
            t = torch.tensor([out.value], dtype=torch.float64, device="cpu" if gloo else a.device)
            dist.all_reduce(t, group=self.halo.group)
            return float(t.item())
        return out.value
