"""Problem validation (RegularizedProblem, reference problem.py:72-75) through
the one-pass device check (csrc/check.cu, adask_check_problem): non-finite A
or B and lam entries that are non-finite or < 1 raise ValueError, as in the
reference; valid inputs pass, for fp64 / fp32, contiguous and strided A."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ak():
    import paper_2104_14101_b200 as ak

    return ak


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("shape", [(1000, 33), (4096, 64), (7, 3)])
def test_valid_problem_passes(ak, dtype, shape):
    n, d = shape
    A = torch.randn(n, d, dtype=dtype, device="cuda")
    p = ak.RegularizedProblem(A, np.ones(d), 0.1, np.full(d, 2.0))
    assert p.n == n and p.d == d


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
@pytest.mark.parametrize("where", [0, 12345, -1])
def test_nonfinite_A_raises(ak, dtype, bad, where):
    A = torch.randn(300, 47, dtype=dtype, device="cuda")
    A.view(-1)[where] = bad
    with pytest.raises(ValueError):
        ak.RegularizedProblem(A, np.ones(47), 0.1)


def test_nonfinite_A_strided_raises(ak):
    full = torch.randn(500, 64, dtype=torch.float64, device="cuda")
    A = full[:, 3:40]
    A[499, 36] = float("nan")
    with pytest.raises(ValueError):
        ak.RegularizedProblem(A, np.ones(37), 0.1)
    A[499, 36] = 1.0
    full[0, 0] = float("nan")  # outside the slice: not part of the problem
    ak.RegularizedProblem(A, np.ones(37), 0.1)


def test_nonfinite_B_raises(ak):
    A = torch.randn(200, 10, dtype=torch.float64, device="cuda")
    B = np.ones(10)
    B[7] = np.inf
    with pytest.raises(ValueError):
        ak.RegularizedProblem(A, B, 0.1)


@pytest.mark.parametrize("lam_bad", [0.5, np.nan, np.inf])
def test_bad_lam_raises(ak, lam_bad):
    A = torch.randn(200, 10, dtype=torch.float64, device="cuda")
    lam = np.full(10, 3.0)
    lam[4] = lam_bad
    with pytest.raises(ValueError):
        ak.RegularizedProblem(A, np.ones(10), 0.1, lam)


def test_validate_false_skips(ak):
    A = torch.randn(200, 10, dtype=torch.float64, device="cuda")
    A[0, 0] = float("nan")
    ak.RegularizedProblem(A, np.ones(10), 0.1, validate=False)
