"""GPU path against the REFERENCE's own outputs (tests/golden/reference_golden.npz):
bit-exact SRHT / SJLT / FWHT, preconditioner and problem kernels within
fp64 tolerance, and the reference's adaptive traces (identical accept /
resketch schedule, x within 1e-8) for the PCG64-driven families."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import recipes as R  # noqa: E402

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz"))


@pytest.fixture(scope="module")
def ak():
    import paper_2104_14101_b200 as ak

    return ak


@pytest.mark.parametrize("i", range(len(R.SRHT_CASES)))
def test_srht_reference_bitwise(ak, i):
    n, d, m, seed = R.SRHT_CASES[i]
    assert np.array_equal(ak.sketch_srht(R.sketch_input("srht", i, n, d), m, seed).SA, G[f"srht{i}_SA"])


@pytest.mark.parametrize("i", range(len(R.SJLT_CASES)))
def test_sjlt_reference_bitwise(ak, i):
    n, d, m, seed = R.SJLT_CASES[i]
    assert np.array_equal(ak.sketch_sjlt(R.sketch_input("sjlt", i, n, d), m, seed).SA, G[f"sjlt{i}_SA"])


@pytest.mark.parametrize("i", range(len(R.SJLT_S_CASES)))
def test_sjlt_s_reference(ak, i):
    n, d, m, seed, s = R.SJLT_S_CASES[i]
    got = ak.sketch_sjlt(R.sketch_input("sjlts", i, n, d), m, seed, s=s).SA
    np.testing.assert_allclose(got, G[f"sjlts{i}_SA"], rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("i", range(len(R.FWHT_CASES)))
def test_fwht_reference_bitwise(ak, i):
    n, d = R.FWHT_CASES[i]
    x = R.sketch_input("fwht", i, n, d)
    assert np.array_equal(ak.fwht(x), G[f"fwht{i}_y"])
    assert np.array_equal(ak.fwht(x, normalized=False), G[f"fwht{i}_yu"])


def test_preconditioner_and_problem_reference(ak):
    pres, (A, B, lam, X) = R.pre_inputs()
    for i, (SA, lamv, Z) in enumerate(pres):
        P = ak.build(SA, 0.7, lamv)
        assert (0 if P.path == "cholesky-d" else 1) == int(G[f"pre{i}_path"][0])
        ref = G[f"pre{i}_out"]
        assert np.linalg.norm(P.solve(Z) - ref) <= 1e-10 * np.linalg.norm(ref)
        np.testing.assert_allclose(P.L, G[f"pre{i}_L"], rtol=1e-10, atol=1e-12)
        dec = ak.approx_newton_decrement(P, Z)
        assert abs(dec - G[f"pre{i}_dec"][0]) <= 1e-10 * abs(G[f"pre{i}_dec"][0])
    p = ak.RegularizedProblem(A, B, 0.8, lam)
    for got, key in ((p.hess_mult(X), "prob_HX"), (p.gradient(X), "prob_grad")):
        assert np.linalg.norm(got - G[key]) <= 1e-13 * np.linalg.norm(G[key])
    xs = ak.direct_solve(p).x_star
    assert np.linalg.norm(xs - G["prob_xstar"]) <= 1e-11 * np.linalg.norm(G["prob_xstar"])


@pytest.mark.parametrize("i", [0, 1, 3])  # PCG64-driven families (the Gaussian uses Philox by design)
def test_adaptive_reference_trace(ak, i):
    method, fam, n, d, decay, nu, lam_u, m0, T = R.RUNS[i]
    A, b, lam = R.run_instance(i)
    p = ak.RegularizedProblem(A, b, nu, lam)
    cfg = ak.AdaptiveConfig.for_method(method, 0.125, m0, T, fam, 1)
    x, tr = ak.adaptive_run(p, np.zeros(d), cfg, method=method, sol=ak.ExactSolution(G[f"run{i}_xstar"]))
    rec = G[f"run{i}_rec"]
    got = np.array([[r.t, r.m, r.k, ["plain", "accepted", "resketch"].index(r.event), r.delta_tilde,
                     r.delta_exact] for r in tr.records])
    assert got.shape == rec.shape
    assert np.array_equal(got[:, :4], rec[:, :4])
    np.testing.assert_allclose(got[:, 4], rec[:, 4], rtol=1e-8, atol=1e-300)
    ref_x = G[f"run{i}_x"]
    assert np.linalg.norm(x - ref_x) <= 1e-8 * np.linalg.norm(ref_x)
