"""Brute-force dense assembly of the 3D Stokes matrix (tier O1).

TEST INFRASTRUCTURE ONLY. Assembles entry (i, j) = a(phi_j, phi_i) of PAPER.md Eq. (3)/(5) under the
symmetric sign [[A, B^T], [B, 0]] cell by cell and face by face with naive per-basis-pair
quadrature, one Gauss point more than the production rule. Shares no code with
oracle/stokes_oracle.cpp (numpy Gauss rules, own Lobatto nodes and Lagrange evaluation). Penalty
gamma = (k+1)(k+2)/h, interior faces gamma [[u]][[v]], boundary 2 gamma u v.
Row/column ordering is the stored level layout: [u_x | u_y | u_z | p], x fastest, with
the boundary-normal DoFs present as zero rows/columns.
"""
import numpy as np
from numpy.polynomial import legendre as npleg


def lobatto_nodes(deg):
    if deg == 0:
        return np.array([0.5])
    c = np.zeros(deg + 1)
    c[-1] = 1.0
    inner = np.sort(npleg.legroots(npleg.legder(c))) if deg > 1 else np.array([])
    return np.concatenate([[0.0], 0.5 * (inner + 1.0), [1.0]])


def lagrange(nodes, x):
    """values and derivatives of the nodal basis at points x: shape (len(nodes), len(x))."""
    x = np.atleast_1d(x)
    nn = len(nodes)
    V = np.ones((nn, len(x)))
    D = np.zeros((nn, len(x)))
    for i in range(nn):
        others = [j for j in range(nn) if j != i]
        for j in others:
            V[i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
        for l in others:
            t = np.full(len(x), 1.0 / (nodes[i] - nodes[l]))
            for j in others:
                if j != l:
                    t *= (x - nodes[j]) / (nodes[i] - nodes[j])
            D[i] += t
    return V, D


class Layout:
    def __init__(self, k, level):
        self.k, self.m = k, 2 << level
        self.n = self.m * (k + 1)
        self.h = 1.0 / self.m
        n = self.n
        self.dims = [[n + 1 if a == c else n for a in range(3)] for c in range(3)]
        self.off = [0, (n + 1) * n * n, 2 * (n + 1) * n * n, 3 * (n + 1) * n * n]
        self.total = self.off[3] + n ** 3

    def vidx(self, c, g):
        d = self.dims[c]
        return self.off[c] + (g[2] * d[1] + g[1]) * d[0] + g[0]

    def pidx(self, g):
        return self.off[3] + (g[2] * self.n + g[1]) * self.n + g[0]


def assemble(k, level):
    L = Layout(k, level)
    m, h, n = L.m, L.h, L.n
    gamma = (k + 1) * (k + 2) / h
    nq = k + 3
    xq, wq = npleg.leggauss(nq)
    xq, wq = 0.5 * (xq + 1.0), 0.5 * wq
    zp, zo = lobatto_nodes(k + 1), lobatto_nodes(k)
    Vp, Dp = lagrange(zp, xq)
    Vo, Do = lagrange(zo, xq)
    ends = np.array([0.0, 1.0])
    Ep, EDp = lagrange(zp, ends)
    Eo, EDo = lagrange(zo, ends)
    A = np.zeros((L.total, L.total))

    def vel_funcs(c, cell):
        """local functions of comp c: list of (global idx or None, (i0,i1,i2))"""
        out = []
        dl = [k + 2 if a == c else k + 1 for a in range(3)]
        for i2 in range(dl[2]):
            for i1 in range(dl[1]):
                for i0 in range(dl[0]):
                    loc = (i0, i1, i2)
                    g = [cell[a] * (k + 1) + loc[a] for a in range(3)]
                    idx = None if g[c] in (0, n) else L.vidx(c, g)
                    out.append((idx, loc))
        return out

    def tabs(c, a):
        return (Vp, Dp) if a == c else (Vo, Do)

    W3 = np.einsum("i,j,k->ijk", wq, wq, wq).ravel(order="F")  # index x fastest
    for ez in range(m):
        for ey in range(m):
            for ex in range(m):
                cell = (ex, ey, ez)
                # values / gradients at quadrature points (x fastest)
                pf = []
                for i2 in range(k + 1):
                    for i1 in range(k + 1):
                        for i0 in range(k + 1):
                            val = np.einsum("i,j,k->ijk", Vo[i0], Vo[i1], Vo[i2]).ravel(order="F")
                            g = [cell[a] * (k + 1) + (i0, i1, i2)[a] for a in range(3)]
                            pf.append((L.pidx(g), val))
                for c in range(3):
                    fs = vel_funcs(c, cell)
                    vals, grads, idxs = [], [], []
                    for idx, loc in fs:
                        T = [tabs(c, a) for a in range(3)]
                        gr = []
                        for d in range(3):
                            f = [T[a][1][loc[a]] if a == d else T[a][0][loc[a]] for a in range(3)]
                            gr.append(np.einsum("i,j,k->ijk", *f).ravel(order="F") / h)
                        idxs.append(idx)
                        grads.append(np.array(gr))
                    for i, gi in zip(idxs, grads):
                        if i is None:
                            continue
                        for j, gj in zip(idxs, grads):
                            if j is None:
                                continue
                            A[i, j] += h ** 3 * np.sum(W3 * np.sum(gi * gj, axis=0))
                        # divergence coupling: (p, d_c v_c) and its transpose
                        for pi, pv in pf:
                            val = h ** 3 * np.sum(W3 * pv * gi[c])
                            A[i, pi] += val
                            A[pi, i] += val
    # faces
    W2 = np.einsum("i,j->ij", wq, wq).ravel(order="F")
    for d in range(3):
        o = [a for a in range(3) if a != d]
        for ez in range(m):
            for ey in range(m):
                for ex in range(m):
                    cell = (ex, ey, ez)
                    for c in range(3):
                        if c == d:
                            continue

                        def traces(cl, side):
                            """functions of comp c in cell cl: value & phys normal-derivative on face at x_d=side"""
                            res = []
                            for idx, loc in vel_funcs(c, cl):
                                if idx is None:
                                    continue
                                T = [tabs(c, a) for a in range(3)]
                                tv = [T[a][0][loc[a]] for a in o]
                                base = np.einsum("i,j->ij", tv[0], tv[1]).ravel(order="F")
                                E, ED = (Ep, EDp) if d == c else (Eo, EDo)
                                res.append((idx, base * E[loc[d], side], base * ED[loc[d], side] / h))
                            return res

                        if cell[d] + 1 < m:  # interior face between cell and cell + e_d
                            nb = list(cell)
                            nb[d] += 1
                            fm, fp = traces(cell, 1), traces(tuple(nb), 0)
                            # jump = u^- - u^+, avg dn = (dn^- + dn^+)/2
                            funcs = [(i, v, dn, +1.0) for i, v, dn in fm] + [(i, v, dn, -1.0) for i, v, dn in fp]
                            for i, vi, di, si in funcs:
                                for j, vj, dj, sj in funcs:
                                    val = gamma * (si * vi) * (sj * vj) - 0.5 * dj * (si * vi) - 0.5 * di * (sj * vj)
                                    A[i, j] += h * h * np.sum(W2 * val)
                        for side in (0, 1):
                            if (side == 0 and cell[d] == 0) or (side == 1 and cell[d] == m - 1):
                                s = 1.0 if side == 1 else -1.0
                                f = traces(cell, side)
                                for i, vi, di in f:
                                    for j, vj, dj in f:
                                        val = 2 * gamma * vi * vj - s * dj * vi - s * di * vj
                                        A[i, j] += h * h * np.sum(W2 * val)
    return A
