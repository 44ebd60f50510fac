"""Harness of the reference (module `harness`): manufactured solution, right-hand
side, L2 errors, divergence, fractional iteration count and a convergence-study driver, on top of the
B200 solver (MG-preconditioned FGMRES, include/smg_b200.h::smg_solve).

This is host-side set-up / post-processing (numpy), not the hot path. Everything is separable on the
unit cube, so the right-hand side is built from 1D integrals (exact tensor structure, no 3D
quadrature) and errors are evaluated on a tensor Gauss grid with k+3 points per cell and direction
(SPEC.md:640).

Manufactured solution (3D): psi = phi(x) phi(y) phi(z),
  u = (psi_y + psi_z, -psi_x - psi_z, -psi_x + psi_y),  p = cos(2 pi x) cos(2 pi y) cos(2 pi z),
  phi(x) = x^2 (x-1)^2 / sqrt(2 pi sigma^2) exp(-(x-mu)^2 / sigma^2),  sigma = 0.1, mu = 0.5,
  f = -Lap u + grad p.
Sign convention: the operator is the symmetric [[A, B^T], [B, 0]] with
B^T p = (p, div v), so the discrete pressure approximates -p; errors compare p_h with -p after
removing both means.
"""
import math
import time

import numpy as np
from numpy.polynomial import legendre as npleg
from numpy.polynomial import polynomial as nppoly


# ---------------------------------------------------------------------------------------------
# 1D ingredients (quadrature.hpp / basis.hpp semantics: nodal Lagrange basis on Gauss-Lobatto points)
# ---------------------------------------------------------------------------------------------
def gauss(n):
    """n-point Gauss rule on [0, 1]."""
    x, w = npleg.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def gauss_lobatto(n):
    """n Gauss-Lobatto points on [0, 1] (endpoints + roots of P'_{n-1})."""
    if n == 1:
        return np.array([0.5])
    c = np.zeros(n)
    c[-1] = 1.0
    inner = npleg.legroots(npleg.legder(c)) if n > 2 else np.array([])
    return np.concatenate([[0.0], 0.5 * (np.sort(inner) + 1.0), [1.0]])


def lagrange(nodes, x, deriv=False):
    """values (or derivatives) of the Lagrange basis on `nodes` at points x: (len(x), len(nodes))."""
    nodes = np.asarray(nodes)
    x = np.asarray(x)
    n = len(nodes)
    V = np.ones((len(x), n))
    if not deriv:
        for i in range(n):
            for j in range(n):
                if j != i:
                    V[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
        return V
    D = np.zeros((len(x), n))
    for i in range(n):
        for mm in range(n):
            if mm == i:
                continue
            t = np.full(len(x), 1.0 / (nodes[i] - nodes[mm]))
            for j in range(n):
                if j != i and j != mm:
                    t *= (x - nodes[j]) / (nodes[i] - nodes[j])
            D[:, i] += t
    return D


def global_basis_at(k, level, continuous, pts_ref, deriv=False):
    """matrix (m * len(pts_ref), n_nodes): global 1D basis (DG degree k, or C0 degree k+1 incl. both
    boundary nodes) at the points pts_ref mapped into every cell (cell-major)."""
    m = 2 << level
    h = 1.0 / m
    deg = k + 1 if continuous else k
    nodes = gauss_lobatto(deg + 1)
    loc = lagrange(nodes, pts_ref, deriv) / (h if deriv else 1.0)
    nq = len(pts_ref)
    nn = m * deg + 1 if continuous else m * (deg + 1)
    B = np.zeros((m * nq, nn))
    for e in range(m):
        c0 = e * deg if continuous else e * (deg + 1)
        B[e * nq:(e + 1) * nq, c0:c0 + deg + 1] += loc
    return B


# ---------------------------------------------------------------------------------------------
# manufactured solution
# ---------------------------------------------------------------------------------------------
class Manufactured:
    """Closed-form phi and its derivatives as (polynomial) * exp(-(x-mu)^2/sigma^2); every field is a
    sum of separable terms coef * a(x) b(y) c(z)."""

    def __init__(self, sigma=0.1, mu=0.5):
        if not sigma > 0:
            raise ValueError("sigma must be > 0")
        self.sigma, self.mu = sigma, mu
        c = 1.0 / math.sqrt(2.0 * math.pi * sigma * sigma)
        P = nppoly.polymul([0, 0, 1.0], nppoly.polymul([-1.0, 1.0], [-1.0, 1.0])) * c  # c x^2 (x-1)^2
        dE = np.array([2.0 * mu / sigma ** 2, -2.0 / sigma ** 2])  # E'/E = -2 (x - mu) / sigma^2
        self.polys = [P]
        for _ in range(4):
            Pn = self.polys[-1]
            self.polys.append(nppoly.polyadd(nppoly.polyder(Pn), nppoly.polymul(Pn, dE)))

    def phi(self, x, d=0):
        x = np.asarray(x, dtype=np.float64)
        return nppoly.polyval(x, self.polys[d]) * np.exp(-((x - self.mu) ** 2) / self.sigma ** 2)

    # separable terms: (coef, (dx, dy, dz)) of phi-derivatives; 'cos' terms for the pressure
    U = {0: [(1.0, (0, 1, 0)), (1.0, (0, 0, 1))],
         1: [(-1.0, (1, 0, 0)), (-1.0, (0, 0, 1))],
         2: [(-1.0, (1, 0, 0)), (1.0, (0, 1, 0))]}

    def u_terms(self, c):
        return [(a, d) for a, d in self.U[c]]

    def lap_terms(self, c):
        out = []
        for a, d in self.U[c]:
            for ax in range(3):
                dd = list(d)
                dd[ax] += 2
                out.append((a, tuple(dd)))
        return out

    @staticmethod
    def cosf(x, d=0):
        """d-th derivative of cos(2 pi x)."""
        w = 2.0 * math.pi
        return [np.cos, lambda t: -np.sin(t), lambda t: -np.cos(t), np.sin][d % 4](w * np.asarray(x)) * w ** d

    def u(self, c, x, y, z):
        return sum(a * self.phi(x, d[0]) * self.phi(y, d[1]) * self.phi(z, d[2]) for a, d in self.U[c])

    def p(self, x, y, z):
        return self.cosf(x) * self.cosf(y) * self.cosf(z)

    def f(self, c, x, y, z):
        """f = -Lap u + grad p."""
        v = -sum(a * self.phi(x, d[0]) * self.phi(y, d[1]) * self.phi(z, d[2]) for a, d in self.lap_terms(c))
        g = [self.cosf(x, c == 0), self.cosf(y, c == 1), self.cosf(z, c == 2)]
        return v + g[0] * g[1] * g[2]

    def div_u(self, x, y, z):
        tot = 0.0
        for c in range(3):
            for a, d in self.U[c]:
                dd = list(d)
                dd[c] += 1
                tot = tot + a * self.phi(x, dd[0]) * self.phi(y, dd[1]) * self.phi(z, dd[2])
        return tot


# ---------------------------------------------------------------------------------------------
# right-hand side and errors on a level (stored layout of include/smg_b200.h: [u_x|u_y|u_z|p])
# ---------------------------------------------------------------------------------------------
def _blocks(v, k, level):
    m = 2 << level
    n = m * (k + 1)
    shapes = []
    for c in range(3):
        d = [n, n, n]
        d[c] = n + 1
        shapes.append((d[2], d[1], d[0]))
    shapes.append((n, n, n))
    out, o = [], 0
    for s in shapes:
        sz = s[0] * s[1] * s[2]
        out.append(v[o:o + sz].reshape(s))
        o += sz
    return out


def assemble_rhs(k, level, ms=None, nq=None):
    """velocity blocks (f_c, phi_i) by per-cell Gauss quadrature of the 1D factors (exact tensor
    structure), constrained boundary-normal entries 0, pressure block 0."""
    ms = ms or Manufactured()
    m = 2 << level
    h = 1.0 / m
    nq = nq or (k + 8)
    qp, qw = gauss(nq)
    X = ((np.arange(m)[:, None] + qp[None, :]) * h).reshape(-1)
    W = np.tile(qw * h, m)
    B = {True: global_basis_at(k, level, True, qp), False: global_basis_at(k, level, False, qp)}
    n = m * (k + 1)
    total = 3 * (n + 1) * n * n + n ** 3
    v = np.zeros(total)
    blk = _blocks(v, k, level)
    for c in range(3):
        F = blk[c]
        terms = [(-a, d, None) for a, d in ms.lap_terms(c)]
        terms.append((1.0, None, c))
        for a, d, gc in terms:
            fac = []
            for ax in range(3):
                g = ms.phi(X, d[ax]) if d is not None else ms.cosf(X, int(ax == gc))
                fac.append(B[ax == c].T @ (W * g))
            F += a * np.einsum("z,y,x->zyx", fac[2], fac[1], fac[0])
        # constrained normal DoFs (planes 0 and n along c)
        idx = [slice(None)] * 3
        for pl in (0, n):
            idx[2 - c] = pl
            F[tuple(idx)] = 0.0
    return v


def l2_errors(k, level, x, ms=None):
    """(err_u, err_p, norm_u, norm_p, div_l2): L2 errors with k+3 Gauss points per cell and
    direction; the pressure is compared as -p_h (symmetric sign) after mean removal; div_l2 is
    ||div u_h||_L2."""
    ms = ms or Manufactured()
    m = 2 << level
    h = 1.0 / m
    qp, qw = gauss(k + 3)
    X = ((np.arange(m)[:, None] + qp[None, :]) * h).reshape(-1)
    W = np.tile(qw * h, m)
    B = {True: global_basis_at(k, level, True, qp), False: global_basis_at(k, level, False, qp)}
    Bd = global_basis_at(k, level, True, qp, deriv=True)
    blk = _blocks(np.asarray(x, dtype=np.float64), k, level)
    Wz = np.einsum("z,y,x->zyx", W, W, W)
    eu = nu = 0.0
    div = 0.0
    for c in range(3):
        M = [B[ax == c] for ax in range(3)]
        uh = np.einsum("zc,yb,xa,cba->zyx", M[2], M[1], M[0], blk[c], optimize=True)
        ue = 0.0
        for a, d in ms.U[c]:
            ue = ue + a * np.einsum("z,y,x->zyx", ms.phi(X, d[2]), ms.phi(X, d[1]), ms.phi(X, d[0]))
        eu += float((Wz * (uh - ue) ** 2).sum())
        nu += float((Wz * ue ** 2).sum())
        Md = list(M)
        Md[c] = Bd
        div = div + np.einsum("zc,yb,xa,cba->zyx", Md[2], Md[1], Md[0], blk[c], optimize=True)
    Bp = B[False]
    ph = -np.einsum("zc,yb,xa,cba->zyx", Bp, Bp, Bp, blk[3], optimize=True)
    pe = np.einsum("z,y,x->zyx", ms.cosf(X), ms.cosf(X), ms.cosf(X))
    ph = ph - (Wz * ph).sum()
    pe = pe - (Wz * pe).sum()
    ep = float((Wz * (ph - pe) ** 2).sum())
    npn = float((Wz * pe ** 2).sum())
    dl2 = float(math.sqrt((Wz * div ** 2).sum()))
    return math.sqrt(eu), math.sqrt(ep), math.sqrt(nu), math.sqrt(npn), dl2


def fractional_count(hist):
    """nu = -8 log10( (||r_n|| / ||r_0||)^(1/n) )."""
    n = len(hist) - 1
    if n < 1 or hist[-1] <= 0:
        return None
    return -8.0 / math.log10((hist[-1] / hist[0]) ** (1.0 / n))


def solve_manufactured(ctx, level, tol=1e-8, max_iter=50, vcycle_precision=None, ms=None):
    """assemble, solve with MG-FGMRES on the device, evaluate: returns a SolveReport dict with the
    columns of SPEC.md:675 (dim, degree, level, dofs, iterations, nu, err_u, err_p, time, dofs/s,
    precision)."""
    import torch

    from . import F32, F64
    vp = F32 if vcycle_precision is None else vcycle_precision
    k = ctx.degree
    b = assemble_rhs(k, level, ms)
    bd = torch.from_numpy(b).to(f"cuda:{ctx.device}")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, it, hist = ctx.solve(level, bd, tol, max_iter, vp)
    torch.cuda.synchronize()
    ts = time.perf_counter() - t0
    eu, ep, nu_, np_, dl2 = l2_errors(k, level, x.cpu().numpy(), ms)
    return {"dim": 3, "degree": k, "level": level, "dofs": int(b.size), "iterations": it,
            "nu": fractional_count(hist), "err_u": eu, "err_p": ep, "rel_err_u": eu / nu_, "rel_err_p": ep / np_,
            "div_l2": dl2, "time_total_s": ts, "dofs_per_s": b.size / ts,
            "precision": "mixed" if vp == F32 else "double", "local_solver": "schur"}


def convergence_study(degrees, levels, tol=1e-8, vcycle_precision=None, device=0, cg_max_iter=30, cg_tol=1e-5):
    """run_convergence_study: one row per (degree, level) plus observed orders."""
    from . import Context
    rows = []
    for k in degrees:
        ctx = Context(k, max(levels), device=device, cg_max_iter=cg_max_iter, cg_tol=cg_tol)
        prev = None
        for level in levels:
            r = solve_manufactured(ctx, level, tol, 60, vcycle_precision)
            if prev is not None:
                r["order_u"] = math.log2(prev["err_u"] / r["err_u"])
                r["order_p"] = math.log2(prev["err_p"] / r["err_p"])
            rows.append(r)
            prev = r
        ctx.close()
    return rows
