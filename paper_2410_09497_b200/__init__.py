"""B200-native hot path of arXiv 2410.09497 (matrix-free multigrid for the H(div)-DG Stokes problem).

Python mirror of the reference's operator / smoother / transfer interface (SPEC.md: apply_stokes,
smooth, prolongate, restrict, v_cycle, fgmres/solve_mixed; BlockVector block_vector.hpp:15-93) over the
C ABI of libsmg_b200.so (include/smg_b200.h). Device vectors are torch CUDA tensors holding one level
vector in the stored layout [u_x | u_y | u_z | p]; torch is used only for device memory and
streams. There is no CPU fallback: if the CUDA library is missing or no sm_100 device is present,
constructing a Context raises.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "libsmg_b200.so")
_LIB = None

SMG_OK, SMG_EINVAL, SMG_ECUDA, SMG_ENOTCONV, SMG_ENOMEM = 0, -22, -100, -101, -12
F64, F32 = 0, 1

EXPORTED = [
    "smg_config_default", "smg_create", "smg_destroy", "smg_set_stream", "smg_last_error", "smg_launch_count",
    "smg_level_sizes", "smg_vec_alloc", "smg_vec_free", "smg_vmult", "smg_residual", "smg_smooth",
    "smg_prolongate_add", "smg_restrict", "smg_coarse_solve", "smg_vcycle", "smg_solve", "smg_dot", "smg_axpy",
    "smg_convert", "smg_vmult_host", "smg_vec_upload", "smg_vec_download", "smg_slab_sizes", "smg_vmult_slab",
    "smg_residual_slab", "smg_dot_slab", "smg_held_sizes", "smg_residual_held", "smg_smooth_colour_held",
    "smg_prolongate_add_held", "smg_restrict_held", "smg_dot_held", "smg_scale", "smg_subtract_from", "smg_norm",
    "smg_project_zero_mean", "smg_pressure_node_weights", "smg_smoother_stats", "smg_nccl_unique_id",
    "smg_dist_init_nccl", "smg_dist_init_transport", "smg_dist_partition", "smg_dist_held", "smg_dist_vmult",
    "smg_dist_dot", "smg_dist_vcycle", "smg_dist_solve",
]


class SmgConfig(ctypes.Structure):
    _fields_ = [("degree", ctypes.c_int), ("max_level", ctypes.c_int), ("device", ctypes.c_int),
                ("cg_max_iter", ctypes.c_int), ("cg_tol", ctypes.c_double), ("cg_fixed", ctypes.c_int),
                ("cg_precond", ctypes.c_int), ("smoother_fused", ctypes.c_int)]


class SmgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"smg error {code}: {msg}")
        self.code = code


class NotConverged(SmgError):
    pass


def build(force=False):
    """Compile libsmg_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(_LIBPATH):
        subprocess.check_call(["make", "-s", "-j8", "-C", _HERE])
    else:
        subprocess.check_call(["make", "-s", "-j8", "-C", _HERE])


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(_LIBPATH):
            raise RuntimeError(f"{_LIBPATH} is missing: run paper_2410_09497_b200.build() (no CPU fallback)")
        L = ctypes.CDLL(_LIBPATH)
        P, I, D, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64
        L.smg_last_error.restype = ctypes.c_char_p
        L.smg_last_error.argtypes = [P]
        L.smg_launch_count.restype = I64
        L.smg_launch_count.argtypes = [P]
        L.smg_create.argtypes = [ctypes.POINTER(SmgConfig), ctypes.POINTER(P)]
        L.smg_destroy.argtypes = [P]
        L.smg_set_stream.argtypes = [P, P]
        L.smg_level_sizes.argtypes = [I, I, P]
        L.smg_vmult.argtypes = [P, I, I, P, P]
        L.smg_residual.argtypes = [P, I, I, P, P, P]
        L.smg_smooth.argtypes = [P, I, I, P, P, I]
        L.smg_prolongate_add.argtypes = [P, I, I, P, P]
        L.smg_restrict.argtypes = [P, I, I, P, P]
        L.smg_coarse_solve.argtypes = [P, I, P, P]
        L.smg_vcycle.argtypes = [P, I, I, P, P]
        L.smg_solve.argtypes = [P, I, P, P, D, I, I, ctypes.POINTER(I), P]
        L.smg_dot.argtypes = [P, I, I, P, P, ctypes.POINTER(D)]
        L.smg_axpy.argtypes = [P, I, I, D, P, P]
        L.smg_convert.argtypes = [P, I, I, P, I, P]
        L.smg_pressure_node_weights.argtypes = [I, P]
        L.smg_smoother_stats.argtypes = [P, I, P, P]
        L.smg_nccl_unique_id.argtypes = [P]
        L.smg_dist_init_nccl.argtypes = [P, P, I, I]
        L.smg_dist_init_transport.argtypes = [P, P, I, I]
        L.smg_dist_partition.argtypes = [I, I, I, P, P]
        L.smg_dist_held.argtypes = [P, I, P, P]
        L.smg_dist_vmult.argtypes = [P, I, I, P, P]
        L.smg_dist_dot.argtypes = [P, I, I, P, P, ctypes.POINTER(D)]
        L.smg_dist_vcycle.argtypes = [P, I, P, P]
        L.smg_dist_solve.argtypes = [P, P, P, D, I, I, ctypes.POINTER(I), P]
        L.smg_scale.argtypes = [P, I, I, D, P]
        L.smg_subtract_from.argtypes = [P, I, I, P, P]
        L.smg_norm.argtypes = [P, I, I, P, ctypes.POINTER(D)]
        L.smg_project_zero_mean.argtypes = [P, I, I, P]
        L.smg_vmult_host.argtypes = [P, I, I, P, P, P, P]
        L.smg_vec_upload.argtypes = [P, I, I, P, P, P]
        L.smg_slab_sizes.argtypes = [I, I, I, I, P]
        L.smg_vmult_slab.argtypes = [P, I, I, P, P, I, I]
        L.smg_residual_slab.argtypes = [P, I, I, P, P, P, I, I]
        L.smg_dot_slab.argtypes = [P, I, I, P, P, I, I, ctypes.POINTER(D)]
        L.smg_held_sizes.argtypes = [I, I, I, I, P]
        L.smg_residual_held.argtypes = [P, I, I, P, P, P, I, I, I, I]
        L.smg_smooth_colour_held.argtypes = [P, I, I, I, P, P, I, I, I, I]
        L.smg_prolongate_add_held.argtypes = [P, I, I, P, P, I, I, I, I, I, I]
        L.smg_restrict_held.argtypes = [P, I, I, P, P, I, I, I, I, I, I]
        L.smg_dot_held.argtypes = [P, I, I, P, P, I, I, I, I, ctypes.POINTER(D)]
        L.smg_vec_download.argtypes = [P, I, I, P, P, P]
        _LIB = L
    return _LIB


def level_sizes(degree, level):
    s = (ctypes.c_int64 * 5)()
    rc = lib().smg_level_sizes(degree, level, s)
    if rc != SMG_OK:
        raise ValueError(f"invalid degree/level ({degree}, {level})")
    return [int(v) for v in s]


def pressure_node_weights(degree):
    """Integrals of the pressure nodal basis over the reference cell (weights of the mass-weighted mean)."""
    w = np.zeros(degree + 1)
    if lib().smg_pressure_node_weights(degree, w.ctypes.data_as(ctypes.c_void_p)) != SMG_OK:
        raise ValueError(f"invalid degree {degree}")
    return w


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """One B200 context for a mesh hierarchy of degree `degree` up to `max_level`.

    Mirrors the reference's per-level operator / smoother / transfer objects (SPEC.md modules
    stokes_op, smoother, multigrid, solver). Methods take torch CUDA tensors (float64 = SMG_F64,
    float32 = SMG_F32) in the stored level layout and launch on torch's current CUDA stream.
    """

    def __init__(self, degree, max_level, device=0, cg_max_iter=30, cg_tol=1e-8, cg_fixed=False, cg_precond=1,
                 smoother_fused=False):
        import torch
        self._torch = torch
        cfg = SmgConfig(degree, max_level, device, cg_max_iter, cg_tol, int(cg_fixed), int(cg_precond),
                        int(smoother_fused))
        h = ctypes.c_void_p()
        rc = lib().smg_create(ctypes.byref(cfg), ctypes.byref(h))
        if rc != SMG_OK:
            msg = lib().smg_last_error(None).decode()
            if rc == SMG_EINVAL:
                raise ValueError(msg)
            raise SmgError(rc, msg)
        self._h = h
        self.degree, self.max_level, self.device = degree, max_level, device
        self._stream = None
        self._sync_stream()

    def close(self):
        if getattr(self, "_h", None):
            lib().smg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- plumbing ----
    def _sync_stream(self):
        s = self._torch.cuda.current_stream(self.device).cuda_stream
        if s != self._stream:
            self._check(lib().smg_set_stream(self._h, ctypes.c_void_p(s)))
            self._stream = s

    def _check(self, rc):
        if rc == SMG_OK:
            return
        msg = lib().smg_last_error(self._h).decode()
        if rc == SMG_EINVAL:
            raise ValueError(msg)
        if rc == SMG_ENOTCONV:
            raise NotConverged(rc, msg)
        raise SmgError(rc, msg)

    def _prec(self, t):
        torch = self._torch
        if not t.is_cuda:
            raise ValueError("device vectors must be CUDA tensors (use vmult_host for host buffers)")
        if not t.is_contiguous():
            raise ValueError("device vectors must be contiguous")
        if t.dtype == torch.float64:
            return F64
        if t.dtype == torch.float32:
            return F32
        raise ValueError("dtype must be float64 or float32")

    def _check_size(self, t, level):
        if t.numel() != self.sizes(level)[4]:
            raise ValueError(f"vector has {t.numel()} entries, level {level} needs {self.sizes(level)[4]}")

    def _vec(self, t, level, prec=None):
        """Validate a device level vector: CUDA, contiguous, on this context's device, float64/float32
        (and equal to `prec` if given), exactly the stored size of `level`. The C ABI takes raw pointers
        without sizes, so a mismatch here would otherwise be an out-of-bounds device access."""
        p = self._prec(t)
        if t.device.index != self.device:
            raise ValueError(f"vector is on cuda:{t.device.index}, the context on cuda:{self.device}")
        if prec is not None and p != prec:
            raise ValueError("all vectors of a call must have the same precision")
        if level < 0 or level > self.max_level:
            raise ValueError(f"level {level} out of range 0..{self.max_level}")
        self._check_size(t, level)
        return p

    def sizes(self, level):
        return level_sizes(self.degree, level)

    def new_vector(self, level, dtype=None):
        torch = self._torch
        return torch.zeros(self.sizes(level)[4], dtype=dtype or torch.float64, device=f"cuda:{self.device}")

    @property
    def launch_count(self):
        return int(lib().smg_launch_count(self._h))

    # ---- hot path ----
    def apply_stokes(self, level, x, out=None):
        """y = A x (apply_stokes)."""
        p = self._vec(x, level)
        y = self._torch.empty_like(x) if out is None else out
        self._vec(y, level, p)
        self._sync_stream()
        self._check(lib().smg_vmult(self._h, level, p, _ptr(y), _ptr(x)))
        return y

    vmult = apply_stokes

    def residual(self, level, b, x, out=None):
        p = self._vec(x, level)
        self._vec(b, level, p)
        r = self._torch.empty_like(x) if out is None else out
        self._vec(r, level, p)
        self._sync_stream()
        self._check(lib().smg_residual(self._h, level, p, _ptr(r), _ptr(b), _ptr(x)))
        return r

    def smooth(self, level, x, b, zero_init=False):
        """one multiplicative colour-by-colour vertex-patch step, in place on x."""
        p = self._vec(x, level)
        self._vec(b, level, p)
        self._sync_stream()
        self._check(lib().smg_smooth(self._h, level, p, _ptr(x), _ptr(b), int(zero_init)))
        return x

    def prolongate_add(self, coarse_level, x_fine, x_coarse):
        p = self._vec(x_fine, coarse_level + 1)
        self._vec(x_coarse, coarse_level, p)
        self._sync_stream()
        self._check(lib().smg_prolongate_add(self._h, coarse_level, p, _ptr(x_fine), _ptr(x_coarse)))
        return x_fine

    def restrict(self, coarse_level, r_fine, out=None):
        p = self._vec(r_fine, coarse_level + 1)
        rc = out if out is not None else self._torch.zeros(self.sizes(coarse_level)[4], dtype=r_fine.dtype,
                                                           device=r_fine.device)
        self._vec(rc, coarse_level, p)
        self._sync_stream()
        self._check(lib().smg_restrict(self._h, coarse_level, p, _ptr(rc), _ptr(r_fine)))
        return rc

    def coarse_solve(self, b):
        p = self._vec(b, 0)
        x = self._torch.zeros_like(b)
        self._sync_stream()
        self._check(lib().smg_coarse_solve(self._h, p, _ptr(x), _ptr(b)))
        return x

    def vcycle(self, level, b):
        p = self._vec(b, level)
        x = self._torch.zeros_like(b)
        self._sync_stream()
        self._check(lib().smg_vcycle(self._h, level, p, _ptr(x), _ptr(b)))
        return x

    def solve(self, level, b, rel_tol=1e-8, max_iter=50, vcycle_precision=F32, allow_not_converged=False):
        """MG-preconditioned FGMRES (solve_mixed SPEC.md:525-533). Returns (x, iterations, history)."""
        if self._vec(b, level) != F64:
            raise ValueError("solve expects a float64 right-hand side")
        x = self._torch.zeros_like(b)
        it = ctypes.c_int()
        hist = np.zeros(max_iter + 1)
        self._sync_stream()
        rc = lib().smg_solve(self._h, level, _ptr(x), _ptr(b), rel_tol, max_iter, vcycle_precision,
                             ctypes.byref(it), hist.ctypes.data_as(ctypes.c_void_p))
        if rc == SMG_ENOTCONV and allow_not_converged:
            rc = SMG_OK
        self._check(rc)
        return x, it.value, hist[: it.value + 1]

    def dot(self, level, a, b):
        p = self._vec(a, level)
        self._vec(b, level, p)
        out = ctypes.c_double()
        self._sync_stream()
        self._check(lib().smg_dot(self._h, level, p, _ptr(a), _ptr(b), ctypes.byref(out)))
        return out.value

    def smoother_stats(self, reset=False):
        """(patches solved, inner Schur-CG iterations) since creation / the last reset."""
        p, it = ctypes.c_int64(), ctypes.c_int64()
        self._sync_stream()
        self._check(lib().smg_smoother_stats(self._h, int(reset), ctypes.byref(p), ctypes.byref(it)))
        return p.value, it.value

    def norm(self, level, x):
        """sqrt(dot(x, x)), fp64 accumulation (norm, block_vector.hpp:63-66)."""
        p = self._vec(x, level)
        out = ctypes.c_double()
        self._sync_stream()
        self._check(lib().smg_norm(self._h, level, p, _ptr(x), ctypes.byref(out)))
        return out.value

    def axpy(self, level, alpha, x, y):
        """y += alpha x (axpy, block_vector.hpp:68-76)."""
        p = self._vec(x, level)
        self._vec(y, level, p)
        self._sync_stream()
        self._check(lib().smg_axpy(self._h, level, p, float(alpha), _ptr(x), _ptr(y)))
        return y

    def scale(self, level, alpha, x):
        """x *= alpha (scale, block_vector.hpp:74-78)."""
        p = self._vec(x, level)
        self._sync_stream()
        self._check(lib().smg_scale(self._h, level, p, float(alpha), _ptr(x)))
        return x

    def subtract_from(self, level, b, y):
        """y = b - y (subtract_from, block_vector.hpp:80-88)."""
        p = self._vec(y, level)
        self._vec(b, level, p)
        self._sync_stream()
        self._check(lib().smg_subtract_from(self._h, level, p, _ptr(b), _ptr(y)))
        return y

    def project_zero_mean(self, level, x):
        """Remove the mass-weighted pressure mean in place (project_zero_mean)."""
        p = self._vec(x, level)
        self._sync_stream()
        self._check(lib().smg_project_zero_mean(self._h, level, p, _ptr(x)))
        return x

    def vmult_host(self, level, x_blocks, precision=F64, out=None):
        """Reference-facing path: host arrays in the BlockVector layout (3 velocity blocks + the pressure
        block in cell-local order; see to_blockvector) in, host arrays out; host<->device
        copies included (block_vector.hpp:17-18)."""
        dt = np.float64 if precision == F64 else np.float32
        s = self.sizes(level)
        xs = [np.ascontiguousarray(a, dtype=dt) for a in x_blocks]
        for i in range(4):
            if xs[i].size != s[i]:
                raise ValueError("block sizes do not match the level layout")
        ys = out if out is not None else [np.empty(s[i], dtype=dt) for i in range(4)]
        for i in range(4):
            if ys[i].size != s[i] or ys[i].dtype != dt or not ys[i].flags.c_contiguous:
                raise ValueError("output blocks do not match the level layout")
        xv = (ctypes.c_void_p * 3)(*[a.ctypes.data for a in xs[:3]])
        yv = (ctypes.c_void_p * 3)(*[a.ctypes.data for a in ys[:3]])
        self._sync_stream()
        self._check(lib().smg_vmult_host(self._h, level, precision, yv, ctypes.c_void_p(ys[3].ctypes.data), xv,
                                         ctypes.c_void_p(xs[3].ctypes.data)))
        return ys


    def upload(self, level, blocks, out=None, dtype=None):
        """BlockVector host blocks (pressure cell-local) -> device level vector (stored layout)."""
        torch = self._torch
        dtype = dtype or (torch.float64 if np.asarray(blocks[0]).dtype == np.float64 else torch.float32)
        prec = F64 if dtype == torch.float64 else F32
        dt = np.float64 if prec == F64 else np.float32
        s = self.sizes(level)
        xs = [np.ascontiguousarray(a, dtype=dt) for a in blocks]
        if any(xs[i].size != s[i] for i in range(4)):
            raise ValueError("block sizes do not match the level layout")
        v = out if out is not None else self.new_vector(level, dtype)
        self._vec(v, level, prec)
        vel = (ctypes.c_void_p * 3)(*[a.ctypes.data for a in xs[:3]])
        self._sync_stream()
        self._check(lib().smg_vec_upload(self._h, level, prec, _ptr(v), vel, ctypes.c_void_p(xs[3].ctypes.data)))
        return v

    def download(self, level, v):
        """device level vector -> BlockVector host blocks (pressure cell-local)."""
        prec = self._vec(v, level)
        dt = np.float64 if prec == F64 else np.float32
        s = self.sizes(level)
        ys = [np.empty(s[i], dtype=dt) for i in range(4)]
        vel = (ctypes.c_void_p * 3)(*[a.ctypes.data for a in ys[:3]])
        self._sync_stream()
        self._check(lib().smg_vec_download(self._h, level, prec, vel, ctypes.c_void_p(ys[3].ctypes.data), _ptr(v)))
        return ys


def pressure_cell_local_index(degree, level):
    """perm such that p_cell_local = p_global_lex[perm] (SPEC.md:174 cell-local pressure numbering)."""
    H = degree + 1
    m = 2 << level
    n = m * H
    c = np.arange(m)
    a = np.arange(H)
    # cell-local index order: cz, cy, cx, az, ay, ax (slowest to fastest)
    gz = (c[:, None, None, None, None, None] * H + a[None, None, None, :, None, None])
    gy = (c[None, :, None, None, None, None] * H + a[None, None, None, None, :, None])
    gx = (c[None, None, :, None, None, None] * H + a[None, None, None, None, None, :])
    return ((gz * n + gy) * n + gx).reshape(-1)


def to_blockvector(v, degree, level):
    """stored level vector (numpy) -> BlockVector blocks [u_x, u_y, u_z, p_cell_local]."""
    b = split_blocks(np.asarray(v), degree, level)
    return [b[0].copy(), b[1].copy(), b[2].copy(), b[3][pressure_cell_local_index(degree, level)]]


def from_blockvector(blocks, degree, level):
    """BlockVector blocks (pressure cell-local) -> stored level vector (numpy)."""
    p = np.empty_like(np.asarray(blocks[3]))
    p[pressure_cell_local_index(degree, level)] = blocks[3]
    return np.concatenate([np.asarray(blocks[0]), np.asarray(blocks[1]), np.asarray(blocks[2]), p])


def split_blocks(v, degree, level):
    """Split a stored level vector into the BlockVector blocks (u_x, u_y, u_z, p)."""
    s = level_sizes(degree, level)
    o = np.cumsum([0] + s[:4])
    return [v[o[i]:o[i + 1]] for i in range(4)]
