"""Harness: manufactured solution identities and RHS / error evaluation on CPU
(through the oracle's FGMRES), and the SPEC acceptance checks on the B200 solver (-m gpu):
optimal L2 convergence (criterion 6), divergence-free solutions (7), mixed precision == double (8),
iteration counts equal to the oracle's."""
import math

import numpy as np
import pytest

import oracle
from paper_2410_09497_b200 import harness as H


def test_manufactured_identities():
    ms = H.Manufactured()
    P = np.random.default_rng(0).uniform(0, 1, (200, 3))
    # div u = 0 (curl construction)
    assert np.abs(ms.div_u(P[:, 0], P[:, 1], P[:, 2])).max() <= 1e-12
    # closed-form derivatives vs central differences (step 1e-6, tol 1e-6 relative)
    x = np.linspace(0.02, 0.98, 41)
    for d in range(4):
        fd = (ms.phi(x + 1e-6, d) - ms.phi(x - 1e-6, d)) / 2e-6
        assert np.abs(fd - ms.phi(x, d + 1)).max() <= 1e-6 * np.abs(ms.phi(x, d + 1)).max()
    # zero trace of u on the boundary and zero-mean pressure
    for c in range(3):
        assert abs(ms.u(c, 0.0, 0.3, 0.7)) < 1e-14 and abs(ms.u(c, 0.4, 1.0, 0.2)) < 1e-14
    q, w = H.gauss(12)
    X = (np.arange(8)[:, None] + q[None, :]).reshape(-1) / 8
    W = np.tile(w / 8, 8)
    assert abs((W * ms.cosf(X)).sum()) < 1e-12
    with pytest.raises(ValueError):
        H.Manufactured(sigma=0.0)


def test_gauss_lobatto_matches_reference_known_values():
    # Appendix B of SURVEY.md (quadrature.hpp gauss_lobatto_points)
    assert np.allclose(H.gauss_lobatto(4), [0, 0.2763932, 0.7236068, 1], atol=1e-7)
    assert np.allclose(H.gauss_lobatto(5), [0, 0.17267316, 0.5, 0.82732684, 1], atol=1e-8)


def test_rhs_and_errors_with_the_oracle_solver():
    # k = 1, levels 1..3 through the CPU oracle: divergence-free discrete solution and decreasing
    # errors; the interpolant-free pipeline (RHS -> solve -> errors) is exercised end to end
    errs = []
    for level in (2, 3):
        b = H.assemble_rhs(1, level)
        x, it, hist = oracle.fgmres(1, level, b, 1e-8, 60, oracle.cg_opts(30, 1e-8, False, 1))
        eu, ep, nu, npn, div = H.l2_errors(1, level, x)
        assert div <= 1e-10 * nu
        errs.append((eu, ep))
    assert math.log2(errs[0][0] / errs[1][0]) >= 1.7  # order 2 for k = 1 (criterion 6)
    assert math.log2(errs[0][1] / errs[1][1]) >= 1.7


@pytest.mark.gpu
def test_gpu_convergence_orders_divergence_mixed():
    import paper_2410_09497_b200 as smg
    rows = {}
    for vp in (smg.F64, smg.F32):
        rows[vp] = H.convergence_study([2], [2, 3, 4], vcycle_precision=vp)
    fine = rows[smg.F64][-1]
    assert fine["order_u"] >= 2.7 and fine["order_p"] >= 2.7  # k + 0.7 (criterion 6)
    for r in rows[smg.F64] + rows[smg.F32]:
        assert r["div_l2"] <= 1e-6 * 1.65e-2  # ||div u_h|| <= 1e-6 ||u_h|| (criterion 7)
    for rd, rm in zip(rows[smg.F64], rows[smg.F32]):  # criterion 8
        assert abs(rm["err_u"] - rd["err_u"]) <= 0.01 * rd["err_u"]
        assert abs(rm["err_p"] - rd["err_p"]) <= 0.01 * rd["err_p"]
        assert rm["iterations"] <= rd["iterations"] + 2


@pytest.mark.gpu
@pytest.mark.parametrize("k,level", [(1, 2), (2, 3)])
def test_gpu_manufactured_iterations_match_oracle(k, level):
    import paper_2410_09497_b200 as smg
    ctx = smg.Context(k, level, cg_max_iter=30, cg_tol=1e-8)
    r = H.solve_manufactured(ctx, level, 1e-8, 60, smg.F64)
    b = H.assemble_rhs(k, level)
    _, it_ref, _ = oracle.fgmres(k, level, b, 1e-8, 60, oracle.cg_opts(30, 1e-8, False, 1))
    assert abs(r["iterations"] - it_ref) <= 1
