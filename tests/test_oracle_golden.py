"""Pin the CPU oracle's 1D layer and mesh/patch semantics to golden vectors generated from the
unmodified reference headers (tests/golden/make_golden.py, /root/reference/proj/include/stokesmg)."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fem1d_golden.json")))


def close(a, b, tol=1e-13):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    scale = max(1.0, np.abs(b).max())
    assert np.abs(a - b).max() <= tol * scale, np.abs(a - b).max()


def test_quadrature_and_lobatto():
    for e in GOLD["quadrature"]:
        p, w = oracle.gauss_quadrature(e["n"])
        close(p, e["points"]); close(w, e["weights"])
    for e in GOLD["lobatto"]:
        close(oracle.gauss_lobatto_points(e["n"]), e["points"])


def test_mass_derivative_penalty():
    for e in GOLD["mass_1d"]:
        close(oracle.mass_matrix_1d(e["da"], e["dt"], e["h"]), e["m"])
    for e in GOLD["derivative_1d"]:
        close(oracle.derivative_matrix_1d(e["dp"], e["dv"]), e["m"])
    for e in GOLD["penalty"]:
        assert abs(oracle.default_penalty(e["k"], e["h"]) - e["value"]) <= 1e-14 * e["value"]


def test_sipg_all_end_conditions():
    for e in GOLD["sipg"]:
        close(oracle.sipg_laplace_1d(e["degree"], e["cells"], e["h"], e["gamma"], e["left"], e["right"]), e["m"],
              tol=2e-13)


def test_global_mass_derivative_embedding():
    for e in GOLD["mass_dg"]:
        close(oracle.mass_matrix_dg(e["degree"], e["cells"], e["h"]), e["m"])
    for e in GOLD["mass_c0"]:
        close(oracle.mass_matrix_c0(e["degree"], e["cells"], e["h"], e["drop"]), e["m"])
    for e in GOLD["derivative_c0"]:
        close(oracle.derivative_matrix_c0(e["pdeg"], e["cells"], e["drop"]), e["m"])
    for e in GOLD["embedding"]:
        close(oracle.embedding_1d(e["degree"], e["continuous"]), e["m"])


def test_spec_known_answers():
    # SPEC.md:110,119 and SURVEY.md Appendix B
    p, w = oracle.gauss_quadrature(2)
    close(p, [0.5 - 0.5 / np.sqrt(3), 0.5 + 0.5 / np.sqrt(3)])
    close(oracle.mass_matrix_1d(1, 1, 1.0), [[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    close(oracle.sipg_laplace_1d(1, 2, 0.5, 12.0, oracle.END_INTERIOR, oracle.END_INTERIOR),
          [[12, 0, -1, 0], [0, 12, -10, -1], [-1, -10, 12, 0], [0, -1, 0, 12]])


def test_patch_enumeration_semantics():
    # mesh.hpp:60-103: x-fastest vertices, colour = sum (v_i mod 2) << i, corner bit i <-> +1 in dir i
    for e in GOLD["patches"]:
        m = 2 << e["level"]
        nv = m - 1
        verts = np.array(e["vertex"]).reshape(-1, 3)
        cells = np.array(e["cells"]).reshape(-1, 8)
        assert len(verts) == nv ** 3
        for i, v in enumerate(verts):
            assert tuple(v) == (1 + i % nv, 1 + (i // nv) % nv, 1 + i // (nv * nv))
            assert e["color"][i] == (v[0] % 2) | ((v[1] % 2) << 1) | ((v[2] % 2) << 2)
            for corner in range(8):
                c = [v[d] - 1 + ((corner >> d) & 1) for d in range(3)]
                assert cells[i, corner] == (c[2] * m + c[1]) * m + c[0]


def test_generalized_eig_against_lapack():
    import scipy.linalg as sla
    for k in (1, 2, 3, 5):
        h = 1.0 / 8
        g = oracle.default_penalty(k, h)
        for L, M in ((oracle.sipg_laplace_1d(k + 1, 2, h, g, 1, 1), oracle.mass_matrix_c0(k + 1, 2, h, True)),
                     (oracle.sipg_laplace_1d(k, 2, h, g, 3, 2), oracle.mass_matrix_dg(k, 2, h))):
            S, lam = oracle.generalized_eig(L, M)
            ref = sla.eigh(L, M, eigvals_only=True)
            close(lam, ref, tol=1e-11)
            close(S.T @ M @ S, np.eye(len(lam)), tol=1e-11)
            close(L @ S, M @ S @ np.diag(lam), tol=1e-10)
            assert lam.min() > 0


def test_oracle_project_zero_mean_kats():
    # constant pressure -> 0; idempotent to 1e-14; mass-weighted mean of the output 0
    import numpy as np
    k, level = 2, 1
    s = oracle.sizes(k, level)
    npr = s[3]
    c = np.zeros(s[4])
    c[-npr:] = 2.5
    assert np.abs(oracle.project_zero_mean(k, level, c)).max() <= 1e-14 * 2.5  # relative to the constant
    x = np.random.default_rng(7).uniform(-1, 1, s[4]) + 0.3
    y = oracle.project_zero_mean(k, level, x)
    assert np.array_equal(y[:-npr], x[:-npr])
    assert np.abs(oracle.project_zero_mean(k, level, y) - y).max() <= 1e-14
    # the weights are the integrals of the nodal basis: a constant's weighted mean is the constant
    n = (2 << level) * (k + 1)
    p = y[-npr:].reshape(n, n, n)
    gl, gw = oracle.gauss_quadrature(k + 2)
    nodes = oracle.gauss_lobatto_points(k + 1)
    w1 = np.array([sum(gw[q] * np.prod([(gl[q] - nodes[j]) / (nodes[a] - nodes[j]) for j in range(k + 1) if j != a])
                       for q in range(k + 2)) for a in range(k + 1)])
    w = w1[np.arange(n) % (k + 1)]
    assert abs(np.einsum("zyx,z,y,x->", p, w, w, w)) <= 1e-13
