"""The DMMA Gram kernels (gram.cu) against plain fp64 numpy:

  dense     SA^T SA + nu^2 diag(lam)           preconditioner.py:70 (and problem.py:109-111)
  woodbury  (SA * (1/lam)) SA^T + nu^2 I       preconditioner.py:72-73

over shapes that exercise every code path: tiles smaller than 128, odd
leading dimensions (the 16-byte packing pass), split-K with the fixed-order
reduction, fp32 operands widened to fp64 (fp32 and fp64 outputs)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ak():
    import paper_2104_14101_b200 as ak

    return ak


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n,d", [(1, 1), (5, 3), (100, 37), (300, 256), (1000, 130), (4096, 1024),
                                 (20000, 300), (2048, 2048), (65536, 512)])
def test_gram_dense_fp64(ak, n, d):
    from paper_2104_14101_b200.preconditioner import gram_dev

    rng = np.random.default_rng(n * 7 + d)
    A = rng.standard_normal((n, d))
    lam = 1.0 + rng.uniform(0, 9, d)
    H = gram_dev(torch.from_numpy(A).cuda(), 0.3, torch.from_numpy(lam).cuda()).cpu().numpy()
    ref = A.T @ A + 0.3 * np.diag(lam)
    assert _rel(H, ref) <= 1e-14
    assert np.array_equal(H, H.T)


@pytest.mark.parametrize("n,d", [(7, 5), (333, 130), (40000, 256)])
def test_gram_dense_fp32_in(ak, n, d):
    from paper_2104_14101_b200.preconditioner import gram_dev
    from paper_2104_14101_b200.problem import gram_fp64

    rng = np.random.default_rng(n + d)
    A = rng.standard_normal((n, d)).astype(np.float32)
    Ad = torch.from_numpy(A).cuda()
    A64 = A.astype(np.float64)
    ref = A64.T @ A64
    # fp64 accumulation of the fp32 entries: fp64-exact up to the fp64 summation
    H64 = gram_fp64(Ad).cpu().numpy()
    assert _rel(H64, ref) <= 1e-14
    # fp32 output: the fp64 result rounded once
    H32 = gram_dev(Ad, 0.0, None).cpu().numpy()
    assert H32.dtype == np.float32
    assert _rel(H32.astype(np.float64), ref) <= 1e-7


@pytest.mark.parametrize("m,d", [(1, 5), (6, 10), (100, 300), (129, 257), (500, 1030), (128, 4096),
                                 (1000, 1024), (2047, 4096)])
def test_gram_woodbury_fp64(ak, m, d):
    from paper_2104_14101_b200.preconditioner import woodbury_gram_dev

    rng = np.random.default_rng(m * 3 + d)
    SA = rng.standard_normal((m, d)) / np.sqrt(m)
    lam = rng.uniform(1, 10, d)
    W = woodbury_gram_dev(torch.from_numpy(SA).cuda(), 0.01, torch.from_numpy(lam).cuda()).cpu().numpy()
    T = SA * (1.0 / lam)[None, :]  # the reference's operand, preconditioner.py:72
    ref = T @ SA.T + 0.01 * np.eye(m)
    assert _rel(W, ref) <= 1e-14


@pytest.mark.parametrize("m,d", [(33, 70), (512, 4096)])
def test_gram_woodbury_fp32(ak, m, d):
    from paper_2104_14101_b200.preconditioner import woodbury_gram_dev

    rng = np.random.default_rng(m + d)
    SA = (rng.standard_normal((m, d)) / np.sqrt(m)).astype(np.float32)
    lam = rng.uniform(1, 10, d)
    W = woodbury_gram_dev(torch.from_numpy(SA).cuda(), 1e-4, torch.from_numpy(lam).cuda()).cpu().numpy()
    S64 = SA.astype(np.float64)
    ref = (S64 * (1.0 / lam)[None, :]) @ S64.T + 1e-4 * np.eye(m)
    assert _rel(W.astype(np.float64), ref) <= 2e-7


def test_gram_deterministic(ak):
    from paper_2104_14101_b200.preconditioner import gram_dev

    rng = np.random.default_rng(11)
    A = torch.from_numpy(rng.standard_normal((30000, 640))).cuda()
    a = gram_dev(A, 0.0, None)
    b = gram_dev(A, 0.0, None)
    assert torch.equal(a, b)


def test_gram_no_library_kernels(ak):
    """libadask links no cuBLAS: the Grams are the repo's own DMMA kernels."""
    import subprocess

    from paper_2104_14101_b200 import _lib

    out = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "cublas" not in out.lower()
