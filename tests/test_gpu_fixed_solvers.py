"""Fixed-sketch solvers through the device path against the REFERENCE's own
runs (tests/golden/fixed_golden.npz, made by make_fixed_golden.py from
/root/reference/pkg/src/adasketch/solvers.py):

  ihs_run         solvers.py:157-190
  pcg_run         solvers.py:193-224   (columnwise, tol early stop)
  polyak_ihs_run  solvers.py:293-328
  cg              solvers.py:104-140

SRHT / SJLT sketches are bit-exact, so the traces must agree record for
record (same length, same m, decrements and exact errors to 1e-9) and the
iterates to 1e-8 (fp64)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from recipes import FIXED_RUNS, fixed_instance  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "fixed_golden.npz"))


@pytest.fixture(scope="module")
def ak():
    import paper_2104_14101_b200 as ak

    return ak


@pytest.mark.parametrize("i", range(len(FIXED_RUNS)))
def test_fixed_solver_matches_reference(ak, i):
    solver, fam, n, d, c, m, rho, seed, T, tol, s = FIXED_RUNS[i]
    A, B, lam, nu = fixed_instance(i)
    p = ak.RegularizedProblem(A, B, nu, lam)
    sol = ak.direct_solve(p)
    x0 = np.zeros((d, c)) if c > 1 else np.zeros(d)
    if solver == "ihs":
        x, tr = ak.ihs_run(p, x0, m, rho, fam, seed, T, sol=sol, s=s)
    elif solver == "pcg":
        x, tr = ak.pcg_run(p, x0, m, fam, seed, T, tol=tol, sol=sol, s=s)
    elif solver == "polyak":
        x, tr = ak.polyak_ihs_run(p, x0, m, rho, fam, seed, T, sol=sol, s=s)
    else:
        x, tr = ak.cg(p, x0, T, tol=tol, sol=sol)
    rec = GOLD[f"f{i}_rec"]
    got = np.array([[r.t, r.m, r.delta_tilde, r.delta_exact] for r in tr.records])
    assert got.shape == rec.shape, (got.shape, rec.shape)
    assert np.array_equal(got[:, 0], rec[:, 0])
    if solver != "cg":
        assert np.array_equal(got[:, 1], rec[:, 1])
    # decrements / exact errors: relative 1e-8, with an absolute floor at the
    # fp64 rounding level of the first record (late records sit near roundoff)
    tol_ = 1e-8 * np.abs(rec[:, 2:]) + 1e-14 * np.abs(rec[0, 2:])
    assert np.all(np.abs(got[:, 2:] - rec[:, 2:]) <= tol_), (got[:, 2:], rec[:, 2:])
    xr = GOLD[f"f{i}_x"]
    assert np.asarray(x).shape == xr.shape
    assert np.linalg.norm(np.asarray(x) - xr) <= 1e-8 * np.linalg.norm(xr)
