"""GPU parity of every libadask kernel against the CPU oracle (oracle/)
on seeded inputs.  Integer/index work and the SRHT/SJLT sketches are
bit-exact; floating-point reductions are checked at the stated tolerances."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import adasketch_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ak():
    import paper_2104_14101_b200 as ak

    return ak


def _dev_integers(seed, first, count, m):
    from paper_2104_14101_b200 import _lib
    from paper_2104_14101_b200 import device as dv

    g = _lib.pcg64_from_seed(seed)
    out = torch.empty(count, dtype=torch.int32, device="cuda")
    nxt = C.c_uint64()
    _lib.check(_lib.lib().adask_pcg64_integers(dv.ctx().handle, C.byref(g), first, count, m,
                                               out.data_ptr(), C.byref(nxt), dv.stream()))
    return out.cpu().numpy().astype(np.int64), int(nxt.value)


@pytest.mark.parametrize("m", [2, 64, 65536, 1, 3, 1000, 2**31 + 1])
def test_pcg64_integers_bit_exact(ak, m):
    n = 20000
    ref = np.random.default_rng(77).integers(0, m, size=n)
    got, nxt = _dev_integers(77, 0, n, m)
    assert np.array_equal(got, ref)


def test_pcg64_integers_offset_and_next(ak):
    # buckets then signs from one stream (embeddings.py:118, 124) for odd n
    n, m = 1001, 3
    rng = np.random.default_rng(5)
    rows = rng.integers(0, m, size=n)
    signs = rng.integers(0, 2, size=n)
    got_rows, nxt = _dev_integers(5, 0, n, m)
    got_signs, _ = _dev_integers(5, nxt, n, 2)
    assert np.array_equal(got_rows, rows)
    assert np.array_equal(got_signs, signs)


def test_philox_gaussian_matches_oracle(ak):
    S = ak.gaussian_matrix(7, 301, seed=2**40 + 17, col0=5).cpu().numpy()
    ref = O.philox_gaussian(7, 301, 2**40 + 17, col0=5)
    np.testing.assert_allclose(S, ref, rtol=1e-14, atol=1e-15)
    assert abs(S.std() * np.sqrt(7) - 1.0) < 0.1


@pytest.mark.parametrize("n,d", [(100, 5), (4096, 256), (1000, 37), (513, 1024), (300, 2048),
                                 (77, 4096), (50, 5000), (1, 3)])
def test_hess_mult_fp64(ak, n, d):
    rng = np.random.default_rng(n * 7 + d)
    A = rng.standard_normal((n, d))
    lam = 1.0 + rng.uniform(0, 3, d)
    B = rng.standard_normal((d, 2))
    X = rng.standard_normal((d, 2))
    p = ak.RegularizedProblem(A, B, 0.3, lam)
    po = O.Problem.make(A, B, 0.3, lam)
    for got, ref in ((p.hess_mult(X), po.hess_mult(X)), (p.gradient(X), po.gradient(X)),
                     (p.hess_mult(X[:, 0]), po.hess_mult(X[:, 0]))):
        assert got.shape == ref.shape
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("n,d", [(1000, 256), (4099, 1024), (300, 4096), (64, 3)])
def test_hess_mult_fp32(ak, n, d):
    rng = np.random.default_rng(d)
    A = rng.standard_normal((n, d)).astype(np.float32)
    X = rng.standard_normal(d)
    p = ak.RegularizedProblem(A, np.zeros(d), 0.5, dtype="float32")
    ref = O.Problem.make(A.astype(np.float64), np.zeros(d), 0.5).hess_mult(X)
    got = p.hess_mult(X)
    # fp32 data: per-thread partials in fp32, cross-thread reduction and accumulation in fp64
    assert np.linalg.norm(got - ref) <= 2e-6 * np.linalg.norm(ref)


@pytest.mark.parametrize("n,d,m,seed", [(64, 5, 16, 9), (1000, 37, 64, 3), (5000, 129, 1000, 4),
                                        (1 << 14, 256, 4096, 5), (20, 8, 1, 2), (333, 16, 333, 8)])
def test_sjlt_bitwise(ak, n, d, m, seed):
    A = np.random.default_rng(seed).standard_normal((n, d))
    got = ak.sketch_sjlt(A, m, seed).SA
    ref = O.sketch_sjlt(A, m, seed)
    assert np.array_equal(got, ref)


def test_sjlt_s_gt_1(ak):
    A = np.random.default_rng(1).standard_normal((200, 6))
    got = ak.sketch_sjlt(A, 16, 25, s=3).SA
    ref = O.sketch_sjlt(A, 16, 25, s=3)
    np.testing.assert_allclose(got, ref, rtol=1e-15, atol=1e-15)
    S = ak.sketch_sjlt(np.eye(30), 16, seed=25, s=3).SA
    assert np.array_equal((S != 0).sum(axis=0), np.full(30, 3))


@pytest.mark.parametrize("n,d,m,seed", [(64, 3, 64, 4), (300, 4, 128, 1), (1000, 7, 500, 2),
                                        (4096, 33, 256, 3), (5000, 17, 3000, 6), (1, 2, 1, 0),
                                        (1 << 16, 8, 32, 11), (70000, 5, 4096, 12)])
def test_srht_bitwise(ak, n, d, m, seed):
    A = np.random.default_rng(seed).standard_normal((n, d))
    got = ak.sketch_srht(A, m, seed).SA
    ref = O.sketch_srht(A, m, seed)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n,d,m,seed", [(4096, 24, 40, 1), (1 << 14, 20, 1 << 14, 2), (65536, 40, 4096, 3),
                                        ((1 << 16) + 32, 17, 513, 4), (1 << 20, 6, 2000, 5), (1 << 21, 3, 3000, 6)])
def test_srht_pipelined_passes_bitwise(ak, n, d, m, seed, monkeypatch):
    """The persistent TMA-pipelined FWHT passes (srht_pipe.cu, forced with
    ADASK_FWHT_PIPE=2) reproduce the reference SRHT bit for bit (fp64),
    including the 10-bit-per-half pass 2 plus last-stage combine at 2^21 rows."""
    monkeypatch.setenv("ADASK_FWHT_PIPE", "2")
    A = np.random.default_rng(seed).standard_normal((n, d))
    got = ak.sketch_srht(A, m, seed).SA
    assert np.array_equal(got, O.sketch_srht(A, m, seed))


@pytest.mark.parametrize("pipe", ["2", "3"])
def test_srht_pipelined_strided_rows(ak, pipe, monkeypatch):
    """A column slice of a wider matrix (lda > d, partial last panel) through
    the pipelined / hybrid passes: bitwise the reference on the slice."""
    from paper_2104_14101_b200.embeddings import srht_dev

    monkeypatch.setenv("ADASK_FWHT_PIPE", pipe)
    full = np.random.default_rng(4).standard_normal((1 << 15, 64))
    Ad = torch.from_numpy(full).cuda()[:, :37]
    got = srht_dev(Ad, 1500, 8).cpu().numpy()
    assert np.array_equal(got, O.sketch_srht(full[:, :37], 1500, 8))


def test_sjlt_streamed_strided_rows(ak, monkeypatch):
    """The streamed SJLT accumulation on a column slice (lda > d): bitwise."""
    from paper_2104_14101_b200.embeddings import sjlt_dev

    monkeypatch.setenv("ADASK_SJLT_PIPE", "2")
    full = np.random.default_rng(6).standard_normal((40000, 96))
    Ad = torch.from_numpy(full).cuda()[:, 16:64]
    got = sjlt_dev(Ad, 512, 13).cpu().numpy()
    assert np.array_equal(got, O.sketch_sjlt(full[:, 16:64], 512, 13))


@pytest.mark.parametrize("n,d,m,seed", [(1 << 16, 40, 4096, 1), (1 << 14, 20, 1 << 14, 2), (4096, 24, 1000, 3),
                                        ((1 << 17) + 32, 16, 2000, 4), (1 << 20, 6, 600, 5)])
def test_srht_hybrid_passes_bitwise(ak, n, d, m, seed, monkeypatch):
    """Pipelined pass 1 + tile-kernel pass 2 (the fp64 many-row default,
    forced with ADASK_FWHT_PIPE=3) reproduces the reference SRHT bit for bit."""
    monkeypatch.setenv("ADASK_FWHT_PIPE", "3")
    A = np.random.default_rng(seed).standard_normal((n, d))
    got = ak.sketch_srht(A, m, seed).SA
    assert np.array_equal(got, O.sketch_srht(A, m, seed))


@pytest.mark.parametrize("n,d,m", [(1 << 16, 64, 64), (1 << 16, 48, 4096), ((1 << 21) - 64, 16, 32768),
                                   (1 << 21, 20, 100)])
def test_srht_pipelined_fp32_matches_tile_kernels(ak, n, d, m, monkeypatch):
    """fp32 data: the pipelined passes run the same butterfly DAG as the tile
    kernels, so the two device paths agree bitwise; both are within fp32
    rounding of the fp64 oracle."""
    from paper_2104_14101_b200.embeddings import srht_dev

    A = torch.randn(n, d, dtype=torch.float32, device="cuda", generator=torch.Generator("cuda").manual_seed(n + m))
    monkeypatch.setenv("ADASK_FWHT_PIPE", "2")
    pipe = srht_dev(A, m, 9)
    monkeypatch.setenv("ADASK_FWHT_PIPE", "0")
    tile = srht_dev(A, m, 9)
    assert torch.equal(pipe, tile)
    if n <= 1 << 16:
        ref = O.sketch_srht(A.double().cpu().numpy(), m, 9)
        assert np.linalg.norm(pipe.double().cpu().numpy() - ref) <= 1e-5 * np.linalg.norm(ref)


@pytest.mark.parametrize("n,d,m,s", [(5000, 34, 300, 1), (70000, 2048, 512, 1), (9000, 64, 4096, 1),
                                     (3000, 48, 40, 3), (20000, 96, 700, 2)])
def test_sjlt_streamed_accumulation_bitwise(ak, n, d, m, s, monkeypatch):
    """The bulk-copy streamed bucket accumulation (sjlt_pipe.cu, forced with
    ADASK_SJLT_PIPE=2) equals the reference's csr product bit for bit."""
    monkeypatch.setenv("ADASK_SJLT_PIPE", "2")
    A = np.random.default_rng(n + m).standard_normal((n, d))
    got = ak.sketch_sjlt(A, m, 17, s=s).SA
    ref = O.sketch_sjlt(A, m, 17, s=s)
    if s == 1:
        assert np.array_equal(got, ref)
    else:
        np.testing.assert_allclose(got, ref, rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("n,d", [(1, 1), (8, 3), (1024, 5), (4096, 2), (1 << 15, 3)])
def test_fwht_bitwise(ak, n, d):
    x = np.random.default_rng(n).standard_normal((n, d))
    assert np.array_equal(ak.fwht(x), O.fwht(x))
    assert np.array_equal(ak.fwht(x, normalized=False), O.fwht(x, normalized=False))


def test_gaussian_sketch_matches_injected_oracle(ak):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((4096, 256))
    for m in (16, 256, 300):
        got = ak.sketch_gaussian(A, m, 1234).SA
        ref = O.sketch_gaussian(A, m, 1234)
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("m,d", [(40, 10), (10, 10), (6, 10), (300, 200), (100, 300), (700, 129)])
def test_precond_solve_both_paths(ak, m, d):
    rng = np.random.default_rng(m + d)
    SA = rng.standard_normal((m, d))
    lam = 1.0 + rng.uniform(0, 2, d)
    nu = 0.7
    P = ak.build(SA, nu, lam)
    Po = O.build(SA, nu, lam)
    assert P.path == Po.path
    Z = rng.standard_normal((d, 3))
    got, ref = P.solve(Z), Po.solve(Z)
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
    np.testing.assert_allclose(P.L, Po.L, rtol=1e-9, atol=1e-12)


def test_cholesky_not_spd(ak):
    from paper_2104_14101_b200.errors import NotPositiveDefinite

    M = np.eye(100)
    M[57, 57] = -1.0
    with pytest.raises(NotPositiveDefinite):
        ak.cholesky(M)
    L = ak.cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]))
    np.testing.assert_allclose(L, [[2.0, 0.0], [1.0, np.sqrt(2.0)]])


@pytest.mark.parametrize("m,d", [(3000, 1030), (1500, 2000), (4096, 1024)])
def test_precond_large(ak, m, d):
    rng = np.random.default_rng(m)
    SA = rng.standard_normal((m, d)) / np.sqrt(m)
    lam = 1.0 + rng.uniform(0, 9, d)
    P = ak.build(SA, 0.05, lam)
    Po = O.build(SA, 0.05, lam)
    z = rng.standard_normal(d)
    got, ref = P.solve(z), Po.solve(z)
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref)


@pytest.mark.parametrize("inv", ["0", "1"])
@pytest.mark.parametrize("m,d", [(40, 31), (50, 33), (100, 65), (300, 97), (900, 700), (2000, 1600)])
def test_precond_inverse_variants(ak, monkeypatch, inv, m, d):
    """Both L^-1 schedules of the cooperative Cholesky (fused row-wise inside
    the factorization; recursive doubling after it) against the oracle."""
    monkeypatch.setenv("ADASK_CHOL_INV", inv)
    rng = np.random.default_rng(m + d)
    SA = rng.standard_normal((m, d)) / np.sqrt(m)
    lam = 1.0 + rng.uniform(0, 9, d)
    P = ak.build(SA, 0.05, lam)
    Po = O.build(SA, 0.05, lam)
    z = rng.standard_normal((d, 2))
    got, ref = P.solve(z), Po.solve(z)
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref)


@pytest.mark.parametrize("k", [1, 63, 64, 65, 700, 2500])
def test_cholesky_sizes(ak, k):
    rng = np.random.default_rng(k)
    X = rng.standard_normal((k + 5, k))
    M = X.T @ X + np.eye(k)
    L = ak.cholesky(M)
    Lo = np.linalg.cholesky(M)
    assert np.linalg.norm(L - Lo) <= 1e-11 * np.linalg.norm(Lo)
    assert np.allclose(np.triu(L, 1), 0.0)


# ---------------------------------------------------------------- TF32 tcgen05 Gaussian sketch
def _tf32_case(n, d, m, row0, seed, accumulate=False):
    from paper_2104_14101_b200.embeddings import gaussian_dev

    rng = np.random.default_rng(n + d + m)
    A = rng.standard_normal((n, d)).astype(np.float32)
    Ad = torch.from_numpy(A).cuda()
    S = O.philox_gaussian(m, n, seed, col0=row0)
    ref = S @ A.astype(np.float64)
    bound = np.abs(S) @ np.abs(A.astype(np.float64))
    base = None
    if accumulate:
        base = torch.from_numpy(rng.standard_normal((m, d)).astype(np.float32)).cuda()
        out = base.clone()
        got = gaussian_dev(Ad, m, seed, row0=row0, tf32=True, out=out, accumulate=True)
        ref = ref + base.cpu().numpy()
    else:
        got = gaussian_dev(Ad, m, seed, row0=row0, tf32=True)
    torch.cuda.synchronize()
    got = got.cpu().numpy().astype(np.float64)
    # tf32 operands (10-bit mantissa, both sides) + fp32 accumulation:
    # |err| <= 2^-9 sum |S||A| elementwise, and ~1e-3 in Frobenius norm
    err = np.abs(got - ref)
    assert np.all(err <= 2.0**-9 * bound + 1e-5), float(np.max(err / (bound + 1e-30)))
    assert np.linalg.norm(got - ref) <= 2e-3 * np.linalg.norm(ref)
    return got


@pytest.mark.parametrize("n,d,m,row0", [(3000, 300, 200, 7), (1000, 64, 128, 0), (777, 516, 4, 3), (777, 513, 5, 3),
                                        (65536, 96, 64, 1 << 33), (20000, 1030, 300, 5),
                                        (4096, 1024, 256, 0), (9000, 2048, 520, 77)])
def test_gaussian_tf32_tcgen05_matches_oracle(n, d, m, row0):
    _tf32_case(n, d, m, row0, seed=99 + n)


def test_gaussian_tf32_accumulate_and_shards():
    _tf32_case(5000, 200, 130, 11, seed=5, accumulate=True)
    # two row shards with global row offsets sum to the whole sketch
    from paper_2104_14101_b200.embeddings import gaussian_dev

    rng = np.random.default_rng(1)
    A = torch.from_numpy(rng.standard_normal((4096, 160)).astype(np.float32)).cuda()
    whole = gaussian_dev(A, 96, 3, tf32=True)
    part = gaussian_dev(A[:2048], 96, 3, tf32=True)
    part = gaussian_dev(A[2048:], 96, 3, row0=2048, tf32=True, out=part, accumulate=True)
    torch.testing.assert_close(part, whole, rtol=0, atol=2e-5)


@pytest.mark.parametrize("k0,mk,m_total,dtype,tf32", [(0, 64, 64, "float64", False), (64, 64, 128, "float64", False),
                                                      (13, 50, 200, "float64", False), (256, 256, 512, "float32", True),
                                                      (6, 30, 64, "float32", True)])
def test_gaussian_rows_offset_matches_oracle(k0, mk, m_total, dtype, tf32):
    from paper_2104_14101_b200.embeddings import gaussian_rows_dev

    rng = np.random.default_rng(k0 + mk)
    n, d = 2000, 96
    A = rng.standard_normal((n, d))
    Ad = torch.from_numpy(A).to("cuda", torch.float32 if dtype == "float32" else torch.float64)
    got = gaussian_rows_dev(Ad, m_total, k0, mk, 11, row0=3, tf32=tf32).double().cpu().numpy()
    S = O.philox_gaussian(m_total, n, 11, col0=3)[k0:k0 + mk]
    Aref = Ad.double().cpu().numpy()
    ref = S @ Aref
    if dtype == "float64":
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    else:
        assert np.all(np.abs(got - ref) <= 2.0**-9 * (np.abs(S) @ np.abs(Aref)) + 1e-5)


def test_repeated_mixed_launches_stress():
    """Ten seconds of random-size dataflow Cholesky factorizations (fp64 /
    fp32, flag epochs and ticket bases carried across launches) interleaved
    with fused SRHT sketches (self-resetting counters, publisher mailboxes),
    each checked against numpy / the oracle (tools/stress_r02.py)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SECONDS="10", SEED="3")
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "stress_r02.py")], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and "stress ok" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]
