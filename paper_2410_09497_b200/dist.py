"""Multi-GPU driver of the C ABI (csrc/dist.cu, include/smg_b200.h smg_dist_*): one Context per GPU /
rank, z-slab partition, the slab V-cycle and MG-preconditioned FGMRES run in C++ inside the library.

The ghost exchange and the reductions go through either
  * NCCL inside the library (init_nccl: rank 0's unique id is broadcast with torch.distributed), or
  * Python callbacks over a torch.distributed group (init_torch_transport) -- gloo on a single-GPU box
    for the multi-process tests: device slices are staged through host memory.
Vectors use the held layout of smg_dist_held (owned cells + 3 ghost layers per interior side).
"""
import ctypes

import numpy as np

from . import F32, F64, SMG_OK, _ptr, lib

EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                               ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                               ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t),
                               ctypes.POINTER(ctypes.c_int), ctypes.c_void_p)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                ctypes.c_void_p)


class Transport(ctypes.Structure):
    _fields_ = [("exchange", EXCHANGE_FN), ("allreduce_sum", ALLREDUCE_FN), ("user", ctypes.c_void_p)]


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        _CUDART = ctypes.CDLL("libcudart.so.12")
        _CUDART.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        _CUDART.cudaStreamSynchronize.argtypes = [ctypes.c_void_p]
    return _CUDART


def partition(level, nranks, rank):
    z0, z1 = ctypes.c_int(), ctypes.c_int()
    if lib().smg_dist_partition(level, nranks, rank, ctypes.byref(z0), ctypes.byref(z1)) != SMG_OK:
        raise ValueError(f"level {level} cannot be split into {nranks} slabs")
    return z0.value, z1.value


class DistContext:
    """The distributed entry points of one rank's Context."""

    def __init__(self, ctx, nranks, rank):
        self.ctx, self.nranks, self.rank = ctx, nranks, rank
        self._keep = None

    # ---- transports ----
    def init_nccl(self, group=None):
        import torch
        import torch.distributed as dist
        buf = (ctypes.c_char * 128)()
        if self.rank == 0:
            self.ctx._check(lib().smg_nccl_unique_id(buf))
        t = torch.tensor(np.frombuffer(bytes(buf), dtype=np.uint8).copy(), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0, group=group)
        uid = (ctypes.c_char * 128).from_buffer_copy(bytes(t.cpu().numpy()))
        self.ctx._check(lib().smg_dist_init_nccl(self.ctx._h, uid, self.nranks, self.rank))
        return self

    def init_torch_transport(self, group=None):
        """callbacks over a torch.distributed group: NCCL groups move the device slices directly (zero-copy
        tensor views of the library's buffers), gloo groups stage them through host memory (tests and
        single-GPU boxes)."""
        import torch
        import torch.distributed as dist
        cr = _cudart()
        if dist.get_backend(group) == "nccl":
            return self._init_torch_nccl_transport(group)

        def exchange(user, nsend, sp, sb, speer, nrecv, rp, rb, rpeer, stream):
            try:
                cr.cudaStreamSynchronize(stream)
                reqs, host_r = [], []
                for i in range(nsend):
                    h = np.empty(sb[i], dtype=np.uint8)
                    cr.cudaMemcpy(h.ctypes.data, sp[i], sb[i], 2)  # device -> host
                    reqs.append(dist.isend(torch.from_numpy(h), int(speer[i]), group=group))
                for i in range(nrecv):
                    h = torch.empty(rb[i], dtype=torch.uint8)
                    host_r.append((h, i))
                    reqs.append(dist.irecv(h, int(rpeer[i]), group=group))
                for q in reqs:
                    q.wait()
                for h, i in host_r:
                    cr.cudaMemcpy(rp[i], h.numpy().ctypes.data, rb[i], 1)  # host -> device
                return 0
            except Exception as e:  # noqa: BLE001 -- reported as a failed transport
                print("exchange callback failed:", e)
                return 1

        def allreduce(user, dev, count, prec, stream):
            try:
                cr.cudaStreamSynchronize(stream)
                dt = np.float64 if prec == F64 else np.float32
                h = np.empty(count, dtype=dt)
                cr.cudaMemcpy(h.ctypes.data, dev, h.nbytes, 2)
                t = torch.from_numpy(h)
                dist.all_reduce(t, group=group)
                cr.cudaMemcpy(dev, t.numpy().ctypes.data, h.nbytes, 1)
                return 0
            except Exception as e:  # noqa: BLE001
                print("allreduce callback failed:", e)
                return 1

        tr = Transport(EXCHANGE_FN(exchange), ALLREDUCE_FN(allreduce), None)
        self._keep = (tr, exchange, allreduce)  # the callbacks must outlive the context
        self.ctx._check(lib().smg_dist_init_transport(self.ctx._h, ctypes.byref(tr), self.nranks, self.rank))
        return self

    def _init_torch_nccl_transport(self, group):
        import torch
        import torch.distributed as dist
        cr = _cudart()
        dev = self.ctx.device

        class _View:  # __cuda_array_interface__ over a raw device pointer: torch views it without a copy
            def __init__(self, ptr, nbytes, typestr="|u1", itemsize=1):
                self.__cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                                 "data": (int(ptr), False), "version": 3}

        def view(ptr, nbytes, typestr="|u1", itemsize=1):
            return torch.as_tensor(_View(ptr, nbytes, typestr, itemsize), device=f"cuda:{dev}")

        def exchange(user, nsend, sp, sb, speer, nrecv, rp, rb, rpeer, stream):
            try:
                cr.cudaStreamSynchronize(stream)
                ops = [dist.P2POp(dist.isend, view(sp[i], sb[i]), int(speer[i]), group) for i in range(nsend)]
                ops += [dist.P2POp(dist.irecv, view(rp[i], rb[i]), int(rpeer[i]), group) for i in range(nrecv)]
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
                torch.cuda.current_stream(dev).synchronize()
                return 0
            except Exception as e:  # noqa: BLE001
                print("exchange callback failed:", e)
                return 1

        def allreduce(user, ptr, count, prec, stream):
            try:
                cr.cudaStreamSynchronize(stream)
                t = view(ptr, count * (8 if prec == F64 else 4), "<f8" if prec == F64 else "<f4", 8 if prec == F64 else 4)
                dist.all_reduce(t, group=group)
                torch.cuda.current_stream(dev).synchronize()
                return 0
            except Exception as e:  # noqa: BLE001
                print("allreduce callback failed:", e)
                return 1

        tr = Transport(EXCHANGE_FN(exchange), ALLREDUCE_FN(allreduce), None)
        self._keep = (tr, exchange, allreduce)
        self.ctx._check(lib().smg_dist_init_transport(self.ctx._h, ctypes.byref(tr), self.nranks, self.rank))
        return self

    def init_single(self):
        """one rank, no transport (the distributed code path on one GPU)."""
        tr = Transport(EXCHANGE_FN(0), ALLREDUCE_FN(0), None)
        self._keep = (tr,)
        self.ctx._check(lib().smg_dist_init_transport(self.ctx._h, ctypes.byref(tr), 1, 0))
        return self

    # ---- layout ----
    def held(self, level):
        cells = (ctypes.c_int * 4)()
        sizes = (ctypes.c_int64 * 5)()
        self.ctx._check(lib().smg_dist_held(self.ctx._h, level, cells, sizes))
        return tuple(cells), [int(v) for v in sizes]

    def extract(self, level, g):
        """held vector of this rank cut from a full-level vector (torch)."""
        import torch
        (z0, z1, zlo, zhi), _ = self.held(level)
        k, H = self.ctx.degree, self.ctx.degree + 1
        n = (2 << level) * H
        full = self.ctx.sizes(level)
        parts, off = [], 0
        for c in range(4):
            plane = (n + 1) * n if c < 2 else n * n
            planes = (zhi - zlo) * H + (1 if c == 2 else 0)
            parts.append(g[off + zlo * H * plane: off + (zlo * H * plane + planes * plane)])
            off += full[c]
        return torch.cat(parts).contiguous()

    def insert_owned(self, level, g, v):
        """write the owned rows of held vector v into the full-level vector g."""
        (z0, z1, zlo, zhi), sizes = self.held(level)
        H = self.ctx.degree + 1
        n = (2 << level) * H
        m = 2 << level
        full = self.ctx.sizes(level)
        goff, hoff = 0, 0
        for c in range(4):
            plane = (n + 1) * n if c < 2 else n * n
            a, b = (z0 - zlo) * H, (z1 - zlo) * H + (1 if c == 2 and z1 == m else 0)
            g[goff + (zlo * H + a) * plane: goff + (zlo * H + b) * plane] = v[hoff + a * plane: hoff + b * plane]
            goff += full[c]
            hoff += sizes[c]
        return g

    # ---- operators ----
    def vmult(self, level, y, x):
        self.ctx._sync_stream()
        self.ctx._check(lib().smg_dist_vmult(self.ctx._h, level, self.ctx._prec(x), _ptr(y), _ptr(x)))
        return y

    def dot(self, level, a, b):
        out = ctypes.c_double()
        self.ctx._sync_stream()
        self.ctx._check(lib().smg_dist_dot(self.ctx._h, level, self.ctx._prec(a), _ptr(a), _ptr(b), ctypes.byref(out)))
        return out.value

    def vcycle(self, b):
        import torch
        x = torch.zeros_like(b)
        self.ctx._sync_stream()
        self.ctx._check(lib().smg_dist_vcycle(self.ctx._h, self.ctx._prec(b), _ptr(x), _ptr(b)))
        return x

    def solve(self, b, rel_tol=1e-8, max_iter=50, vcycle_precision=F32):
        import torch
        x = torch.zeros_like(b)
        it = ctypes.c_int()
        hist = np.zeros(max_iter + 1)
        self.ctx._sync_stream()
        self.ctx._check(lib().smg_dist_solve(self.ctx._h, _ptr(x), _ptr(b), rel_tol, max_iter, vcycle_precision,
                                             ctypes.byref(it), hist.ctypes.data_as(ctypes.c_void_p)))
        return x, it.value, hist[: it.value + 1]
