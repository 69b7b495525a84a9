"""GPU adaptive solvers vs the CPU oracle: identical sketch-size schedule
(every accept / resketch decision) and final x within 1e-8 (fp64)."""
import numpy as np
import pytest

from oracle import adasketch_oracle as O

pytestmark = pytest.mark.gpu


def _instance(n, d, sigma, nu, lam_uniform, seed=0):
    A, b, lam = O.make_config_problem(n, d, sigma, nu, lam_uniform, data_seed=seed)
    return A, b, lam


def _run_both(method, family, A, b, lam, nu, m_init, T, seed=1, rho=0.125):
    import paper_2104_14101_b200 as ak

    p = ak.RegularizedProblem(A, b, nu, lam)
    cfg = ak.AdaptiveConfig.for_method(method, rho, m_init, T, family, seed)
    x, tr = ak.adaptive_run(p, np.zeros(A.shape[1]), cfg, method=method)
    po = O.Problem.make(A, b, nu, lam)
    xo, tro = O.adaptive_run(po, np.zeros(A.shape[1]), method, rho, m_init, T, family, seed)
    return x, tr, xo[:, 0], tro


def _events(tr):
    return [(r.t, r.m, r.k, r.event) for r in tr.records]


def test_adaptive_ihs_gaussian_cfg0_shape():
    j = np.arange(1, 257, dtype=float)
    A, b, lam = _instance(4096, 256, j**-1.0, 1e-1, False)
    x, tr, xo, tro = _run_both("ihs", "gaussian", A, b, lam, 1e-1, 16, 10)
    assert _events(tr) == _events(tro)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_adaptive_pcg_srht_small():
    j = np.arange(1, 129, dtype=float)
    A, b, lam = _instance(1 << 12, 128, 0.98**j, 1e-2, False)
    x, tr, xo, tro = _run_both("pcg", "srht", A, b, lam, 1e-2, 8, 8)
    assert _events(tr) == _events(tro)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_adaptive_pcg_sjlt_small_lam():
    j = np.arange(1, 129, dtype=float)
    A, b, lam = _instance(1 << 13, 128, j**-0.5, 1e-3, True)
    x, tr, xo, tro = _run_both("pcg", "sjlt", A, b, lam, 1e-3, 8, 8)
    assert _events(tr) == _events(tro)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_direct_solve_and_exact_error():
    import paper_2104_14101_b200 as ak

    rng = np.random.default_rng(4)
    A = rng.standard_normal((500, 40))
    B = rng.standard_normal((40, 2))
    lam = 1.0 + rng.uniform(0, 2, 40)
    p = ak.RegularizedProblem(A, B, 0.8, lam)
    po = O.Problem.make(A, B, 0.8, lam)
    xs = ak.direct_solve(p).x_star
    xso = O.direct_solve(po)
    assert np.linalg.norm(xs - xso) <= 1e-12 * np.linalg.norm(xso)
    x = rng.standard_normal((40, 2))
    e = ak.exact_error(p, x, ak.ExactSolution(xso))
    eo = O.exact_error(po, x, xso)
    assert abs(e - eo) <= 1e-12 * abs(eo)
