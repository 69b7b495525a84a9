"""Pin the CPU oracle (oracle/adasketch_oracle.py) against outputs of the
reference implementation itself (tests/golden/reference_golden.npz, made by
tests/golden/make_golden.py from /root/reference).  CPU only."""
import os
import sys

import numpy as np
import pytest

from oracle import adasketch_oracle as O

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import recipes as R  # noqa: E402

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz"))


def test_derive_seed():
    for (b, k), v in zip(G["derive_in"], G["derive_out"]):
        assert O.derive_seed(int(b), int(k)) == int(v)


@pytest.mark.parametrize("i", range(len(R.SRHT_CASES)))
def test_srht_bitwise(i):
    n, d, m, seed = R.SRHT_CASES[i]
    A = R.sketch_input("srht", i, n, d)
    assert np.array_equal(O.sketch_srht(A, m, seed), G[f"srht{i}_SA"])
    bits, idx = O.srht_draws(n, m, seed)
    assert np.array_equal(bits, G[f"srht{i}_bits"]) and np.array_equal(idx, G[f"srht{i}_idx"])


@pytest.mark.parametrize("i", range(len(R.SJLT_CASES)))
def test_sjlt_bitwise(i):
    n, d, m, seed = R.SJLT_CASES[i]
    A = R.sketch_input("sjlt", i, n, d)
    assert np.array_equal(O.sketch_sjlt(A, m, seed), G[f"sjlt{i}_SA"])
    assert np.array_equal(O.sjlt_sequential(A, m, seed), G[f"sjlt{i}_SA"])  # ascending per-bucket sums
    rows, bits = O.sjlt_draws(n, m, seed)
    assert np.array_equal(rows, G[f"sjlt{i}_rows"]) and np.array_equal(bits, G[f"sjlt{i}_bits"])


@pytest.mark.parametrize("i", range(len(R.SJLT_S_CASES)))
def test_sjlt_s(i):
    n, d, m, seed, s = R.SJLT_S_CASES[i]
    A = R.sketch_input("sjlts", i, n, d)
    assert np.array_equal(O.sketch_sjlt(A, m, seed, s), G[f"sjlts{i}_SA"])


@pytest.mark.parametrize("i", range(len(R.FWHT_CASES)))
def test_fwht(i):
    n, d = R.FWHT_CASES[i]
    x = R.sketch_input("fwht", i, n, d)
    assert np.array_equal(O.fwht(x), G[f"fwht{i}_y"])
    assert np.array_equal(O.fwht(x, normalized=False), G[f"fwht{i}_yu"])


def test_preconditioner_and_problem():
    pres, (A, B, lam, X) = R.pre_inputs()
    for i, (SA, lamv, Z) in enumerate(pres):
        P = O.build(SA, 0.7, lamv)
        assert (0 if P.path == "cholesky-d" else 1) == int(G[f"pre{i}_path"][0])
        np.testing.assert_allclose(P.solve(Z), G[f"pre{i}_out"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(P.L, G[f"pre{i}_L"], rtol=1e-12, atol=1e-13)
    p = O.Problem.make(A, B, 0.8, lam)
    np.testing.assert_allclose(p.hess_mult(X), G["prob_HX"], rtol=1e-13)
    np.testing.assert_allclose(p.gradient(X), G["prob_grad"], rtol=1e-12, atol=1e-12)
    xs = O.direct_solve(p)
    np.testing.assert_allclose(xs, G["prob_xstar"], rtol=1e-12)
    assert abs(O.exact_error(p, X, xs) - G["prob_err"][0]) <= 1e-12 * G["prob_err"][0]


@pytest.mark.parametrize("i", range(len(R.RUNS)))
def test_adaptive_trace(i):
    method, fam, n, d, decay, nu, lam_u, m0, T = R.RUNS[i]
    A, b, lam = R.run_instance(i)
    p = O.Problem.make(A, b, nu, lam)
    sk = O.numpy_gaussian if fam == "gaussian" else None
    x, tr = O.adaptive_run(p, np.zeros(d), method, 0.125, m0, T, fam, 1, x_star=G[f"run{i}_xstar"],
                           sketcher=sk)
    rec = G[f"run{i}_rec"]
    got = np.array([[r.t, r.m, r.k, ["plain", "accepted", "resketch"].index(r.event), r.delta_tilde,
                     r.delta_exact] for r in tr.records])
    assert got.shape == rec.shape
    assert np.array_equal(got[:, :4], rec[:, :4])  # identical accept / resketch schedule
    np.testing.assert_allclose(got[:, 4], rec[:, 4], rtol=1e-9, atol=1e-300)
    np.testing.assert_allclose(x[:, 0], G[f"run{i}_x"], rtol=1e-10, atol=1e-14)
