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


# ---- fp64 Gaussian sketch on the FP64 tensor cores (gauss.cu -> gemm_tn_tc):
# S^T chunks (Philox, transposed) times the rows of A, embeddings.py:66-73
@pytest.mark.parametrize("n,d,m", [(1, 2, 1), (37, 6, 5), (2000, 96, 50), (4096, 256, 16), (4096, 256, 300),
                                   (20000, 130, 129), (65536, 384, 260)])
def test_gaussian_fp64_dmma_matches_injected_oracle(ak, n, d, m):
    from oracle import adasketch_oracle as O
    from paper_2104_14101_b200.embeddings import gaussian_dev

    rng = np.random.default_rng(n + 3 * d + m)
    A = rng.standard_normal((n, d))
    got = gaussian_dev(torch.from_numpy(A).cuda(), m, 77, row0=5).cpu().numpy()
    S = O.philox_gaussian(m, n, 77, col0=5)
    ref = S @ A
    assert _rel(got, ref) <= 1e-13
    # elementwise: fp64 accumulation error only
    assert np.all(np.abs(got - ref) <= 1e-13 * (np.abs(S) @ np.abs(A)) + 1e-300)


def test_gaussian_fp64_dmma_shards_and_pipe_variant(ak, monkeypatch):
    """Row shards accumulate to the whole sketch, and the FP64-pipe GEMM
    (unaligned rows of A take it) agrees with the DMMA path."""
    from paper_2104_14101_b200.embeddings import gaussian_dev

    rng = np.random.default_rng(9)
    A = torch.from_numpy(rng.standard_normal((6000, 200))).cuda()
    whole = gaussian_dev(A, 72, 3)
    part = gaussian_dev(A[:2500].contiguous(), 72, 3)
    part = gaussian_dev(A[2500:].contiguous(), 72, 3, row0=2500, out=part, accumulate=True)
    torch.testing.assert_close(part, whole, rtol=0, atol=1e-12)
    # odd leading dimension: rows not 16-byte aligned -> FP64-pipe path
    Ao = torch.empty((6000, 201), dtype=torch.float64, device="cuda")[:, :200]
    Ao.copy_(A)
    assert Ao.stride(0) == 201
    pipe = gaussian_dev(Ao, 72, 3)
    torch.testing.assert_close(pipe, whole, rtol=0, atol=1e-12)


def test_gaussian_fp64_uses_dmma_kernel(ak):
    """The fp64 Gaussian launches the repo's DMMA GEMM (profiler kernel names)."""
    from torch.profiler import ProfilerActivity, profile

    from paper_2104_14101_b200.embeddings import gaussian_dev

    A = torch.randn((8192, 256), dtype=torch.float64, device="cuda")
    gaussian_dev(A, 64, 1)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        gaussian_dev(A, 64, 1)
        torch.cuda.synchronize()
    names = [e.key for e in prof.key_averages()]
    assert any("k_gemm_tn_dmma" in k for k in names), names
    assert not any(("cutlass" in k or "cublas" in k.lower() or "gemm_kernel" in k) for k in names), names
