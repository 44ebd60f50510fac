"""CPU oracle (TEST INFRASTRUCTURE ONLY).

ctypes wrapper over oracle/liboracle.so, the CPU restatement of the reference algorithm
(see oracle/stokes_oracle.h). Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

END_NONE, END_STRONG, END_NITSCHE, END_INTERIOR = 0, 1, 2, 3


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE], stdout=subprocess.DEVNULL)


def build_native():
    """-march=native build for the timed CPU-baseline legs (the reference's Release flags,
    proj/CMakeLists.txt:26-27); compiled on the host that runs it, into oracle/_native/."""
    subprocess.check_call(["make", "-s", "-C", _HERE, "native"], stdout=subprocess.DEVNULL)


def use_native():
    """Load the -march=native build instead of the portable one (call before the first lib())."""
    global _NATIVE
    _NATIVE = True


_NATIVE = False


def lib():
    global _LIB
    if _LIB is None:
        if _NATIVE:
            build_native()
            path = os.path.join(_HERE, "_native", "liboracle.so")
        else:
            path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        _LIB = ctypes.CDLL(path)
        d, i, i64 = ctypes.c_double, ctypes.c_int, ctypes.c_int64
        P = ctypes.c_void_p
        _LIB.orc_default_penalty.restype = d
        _LIB.orc_default_penalty.argtypes = [i, d]
        _LIB.orc_sipg_laplace_1d.argtypes = [i, i, d, d, i, i, P, i, P, P]
        _LIB.orc_mass_matrix_1d.argtypes = [i, i, d, P, i, P, P]
        _LIB.orc_mass_matrix_dg.argtypes = [i, i, d, P, i, P, P]
        _LIB.orc_mass_matrix_c0.argtypes = [i, i, d, i, P, i, P, P]
        _LIB.orc_sizes.argtypes = [i, i, P]
        _LIB.orc_fgmres.argtypes = [i, i, P, P, d, i, P, P]
        _LIB.orc_set_threads.argtypes = [i]
    return _LIB


class CGOpts(ctypes.Structure):
    _fields_ = [("cg_max_iter", ctypes.c_int), ("cg_tol", ctypes.c_double), ("cg_fixed", ctypes.c_int),
                ("cg_precond", ctypes.c_int)]


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _mat(fn, *args):
    buf = np.zeros(1 << 16)
    r, c = ctypes.c_int(), ctypes.c_int()
    rc = fn(*args, _ptr(buf), ctypes.c_int(buf.size), ctypes.byref(r), ctypes.byref(c))
    if rc != 0:
        raise ValueError(f"oracle call failed ({rc})")
    return buf[: r.value * c.value].reshape(r.value, c.value).copy()


def gauss_quadrature(n):
    p, w = np.zeros(n), np.zeros(n)
    if lib().orc_gauss_quadrature(n, _ptr(p), _ptr(w)) != 0:
        raise ValueError("n must be >= 1")
    return p, w


def gauss_lobatto_points(n):
    p = np.zeros(max(n, 1))
    if lib().orc_gauss_lobatto_points(n, _ptr(p)) != 0:
        raise ValueError("need >= 2 points")
    return p


def mass_matrix_1d(deg_ansatz, deg_test, h):
    return _mat(lib().orc_mass_matrix_1d, deg_ansatz, deg_test, ctypes.c_double(h))


def derivative_matrix_1d(deg_p, deg_v):
    return _mat(lib().orc_derivative_matrix_1d, deg_p, deg_v)


def sipg_laplace_1d(degree, cells, h, gamma, left, right):
    return _mat(lib().orc_sipg_laplace_1d, degree, cells, ctypes.c_double(h), ctypes.c_double(gamma), left, right)


def mass_matrix_dg(degree, cells, h):
    return _mat(lib().orc_mass_matrix_dg, degree, cells, ctypes.c_double(h))


def mass_matrix_c0(degree, cells, h, drop):
    return _mat(lib().orc_mass_matrix_c0, degree, cells, ctypes.c_double(h), int(drop))


def derivative_matrix_c0(pdeg, cells, drop):
    return _mat(lib().orc_derivative_matrix_c0, pdeg, cells, int(drop))


def embedding_1d(degree, continuous):
    return _mat(lib().orc_embedding_1d, degree, int(continuous))


def default_penalty(k, h):
    return lib().orc_default_penalty(k, h)


def generalized_eig(L, M):
    n = L.shape[0]
    L = np.ascontiguousarray(L, dtype=np.float64)
    M = np.ascontiguousarray(M, dtype=np.float64)
    S, lam = np.zeros((n, n)), np.zeros(n)
    if lib().orc_generalized_eig(n, _ptr(L), _ptr(M), _ptr(S), _ptr(lam)) != 0:
        raise ValueError("generalized_eig failed")
    return S, lam


def sizes(k, level):
    s = np.zeros(5, dtype=np.int64)
    lib().orc_sizes(k, level, _ptr(s))
    return [int(v) for v in s]


def cg_opts(max_iter=30, tol=1e-12, fixed=True, precond=1):
    return CGOpts(max_iter, tol, int(fixed), int(precond))


def apply_stokes(k, level, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    if lib().orc_apply_stokes(k, level, _ptr(x), _ptr(y)) != 0:
        raise ValueError("apply_stokes failed")
    return y


def residual(k, level, b, x):
    r = np.zeros_like(b)
    lib().orc_residual(k, level, _ptr(np.ascontiguousarray(b)), _ptr(np.ascontiguousarray(x)), _ptr(r))
    return r


def smooth(k, level, x, b, opts=None):
    opts = opts or cg_opts()
    x = np.array(x, dtype=np.float64, copy=True)
    it = ctypes.c_int()
    if lib().orc_smooth(k, level, _ptr(x), _ptr(np.ascontiguousarray(b)), ctypes.byref(opts), ctypes.byref(it)):
        raise ValueError("smooth failed")
    return x, it.value


def patch_sizes(k):
    s = (ctypes.c_int * 4)()
    lib().orc_patch_sizes(k, s)
    return list(s)


def patch_solve(k, level, vertex, F, G, opts=None):
    opts = opts or cg_opts()
    sz = patch_sizes(k)
    U, P = np.zeros(3 * sz[0]), np.zeros(sz[3])
    v = (ctypes.c_int * 3)(*vertex)
    it = ctypes.c_int()
    rc = lib().orc_patch_solve(k, level, v, _ptr(np.ascontiguousarray(F)), _ptr(np.ascontiguousarray(G)),
                               _ptr(U), _ptr(P), ctypes.byref(opts), ctypes.byref(it))
    if rc:
        raise ValueError("patch_solve failed")
    return U, P, it.value


def prolongate_add(k, coarse_level, xc, xf):
    xf = np.array(xf, dtype=np.float64, copy=True)
    lib().orc_prolongate_add(k, coarse_level, _ptr(np.ascontiguousarray(xc)), _ptr(xf))
    return xf


def restrict(k, coarse_level, rf):
    rc = np.zeros(sizes(k, coarse_level)[4])
    lib().orc_restrict(k, coarse_level, _ptr(np.ascontiguousarray(rf)), _ptr(rc))
    return rc


def coarse_solve(k, b):
    x = np.zeros_like(b)
    lib().orc_coarse_solve(k, _ptr(np.ascontiguousarray(b)), _ptr(x))
    return x


def vcycle(k, level, b, opts=None):
    opts = opts or cg_opts()
    x = np.zeros_like(b)
    lib().orc_vcycle(k, level, _ptr(np.ascontiguousarray(b)), _ptr(x), ctypes.byref(opts))
    return x


def fgmres(k, level, b, tol=1e-8, max_iter=50, opts=None):
    opts = opts or cg_opts()
    x = np.zeros_like(b)
    hist = np.zeros(max_iter + 1)
    it = lib().orc_fgmres(k, level, _ptr(np.ascontiguousarray(b)), _ptr(x), tol, max_iter, ctypes.byref(opts),
                          _ptr(hist))
    if it < 0:
        raise ValueError("fgmres failed")
    return x, it, hist[: it + 1]


def project_zero_mean(k, level, x):
    """Mass-weighted pressure mean removal (project_zero_mean)."""
    x = np.array(x, dtype=np.float64, copy=True)
    if lib().orc_project_zero_mean(k, level, _ptr(x)) != 0:
        raise ValueError("project_zero_mean failed")
    return x


def apply_stokes_sample(k, level, x, z0, z1, y=None):
    """Timing sample: the operator on the cells z in [z0, z1) (rows at the ends incomplete)."""
    y = np.zeros_like(x) if y is None else y
    if lib().orc_apply_stokes_sample(k, level, _ptr(x), _ptr(y), int(z0), int(z1)) != 0:
        raise ValueError("apply_stokes_sample failed")
    return y


def smooth_sample(k, level, x, b, vz0, vz1, opts=None):
    """Timing sample: one smoothing step on the patches with vertex z plane in [vz0, vz1], in place."""
    opts = opts or cg_opts()
    it = ctypes.c_int()
    if lib().orc_smooth_sample(k, level, _ptr(x), _ptr(b), ctypes.byref(opts), int(vz0), int(vz1), ctypes.byref(it)):
        raise ValueError("smooth_sample failed")
    return it.value


def set_threads(n):
    lib().orc_set_threads(int(n))


def constrained_mask(k, level):
    """Boolean mask of the constrained boundary-normal DoFs in the stored level layout."""
    s = sizes(k, level)
    n = (2 << level) * (k + 1)
    mask = np.zeros(s[4], dtype=bool)
    off = 0
    for c in range(3):
        dims = [n + 1 if a == c else n for a in range(3)]
        arr = np.zeros(dims[::-1], dtype=bool)  # (z, y, x)
        sl = [slice(None)] * 3
        sl[2 - c] = 0
        arr[tuple(sl)] = True
        sl[2 - c] = n
        arr[tuple(sl)] = True
        mask[off:off + arr.size] = arr.ravel()
        off += arr.size
    return mask
