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


def test_block_srht_sketcher_bitwise():
    import torch

    import paper_2104_14101_b200 as ak
    from paper_2104_14101_b200.embeddings import SketchSpec
    from paper_2104_14101_b200.parallel import block_srht_sketcher

    rng = np.random.default_rng(9)
    A = rng.standard_normal((5 * 512 + 100, 6))
    p = ak.RegularizedProblem(A, np.zeros(6), 0.1)
    SA = block_srht_sketcher(512)(p, SketchSpec("srht-block", 64, 77)).cpu().numpy()
    assert np.array_equal(SA, O.block_srht(A, 64, 77, 512))


def test_sharded_problem_allreduce_hook_world1():
    """The allreduce hook inside the fused iteration bodies (NCCL, world 1):
    same schedule and x as the unsharded solver."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    import paper_2104_14101_b200 as ak
    from paper_2104_14101_b200.parallel import Comm, ShardedProblem, shard_rows, sharded_sketcher

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        j = np.arange(1, 129, dtype=float)
        A, b, lam = _instance(1 << 13, 128, j**-0.5, 1e-3, True)
        comm = Comm()
        comm.world = 2  # force the exchange path (all-reduce over the single rank)
        plan = shard_rows(A.shape[0], 1, 0)
        ps = ShardedProblem(A, b, 1e-3, lam, plan=plan, comm=comm)
        cfg = ak.AdaptiveConfig.for_method("pcg", 0.125, 8, 8, "sjlt", 1)
        x, tr = ak.adaptive_run(ps, np.zeros(128), cfg, sketcher=sharded_sketcher(comm))
        p = ak.RegularizedProblem(A, b, 1e-3, lam)
        x1, tr1 = ak.adaptive_run(p, np.zeros(128), cfg)
        assert _events(tr) == _events(tr1)
        assert np.linalg.norm(x - x1) <= 1e-10 * np.linalg.norm(x1)
        # the native driver on the sharded problem: the all-reduce hook inside
        # the two-column proposal pass (restart reuse) and the sketches
        for method in ("pcg", "ihs"):
            cfg_m = ak.AdaptiveConfig.for_method(method, 0.125, 8, 8, "sjlt", 1)
            xn, trn = ak.adaptive_run(ps, np.zeros(128), cfg_m, method=method, native=True)
            xr, trr = ak.adaptive_run(p, np.zeros(128), cfg_m, method=method)
            assert _events(trn) == _events(trr)
            assert np.linalg.norm(xn - xr) <= 1e-10 * np.linalg.norm(xr)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("method,family", [("pcg", "srht"), ("pcg", "sjlt"), ("ihs", "gaussian"),
                                           ("ihs", "sjlt"), ("pcg", "srht-block")])
def test_native_driver_matches_python_driver(method, family):
    """adask_adaptive_run (C++) and the Python loop run the same kernels in the
    same order: identical traces, bitwise."""
    import paper_2104_14101_b200 as ak

    j = np.arange(1, 97, dtype=float)
    A, b, lam = _instance(4096, 96, j**-0.5, 1e-2, True)
    p = ak.RegularizedProblem(A, b, 1e-2, lam)
    sol = ak.direct_solve(p)
    cfg = ak.AdaptiveConfig.for_method(method, 0.125, 4, 7, family, 3)
    x1, t1 = ak.adaptive_run(p, np.zeros(96), cfg, method=method, sol=sol, native=True, block=1024)
    x2, t2 = ak.adaptive_run(p, np.zeros(96), cfg, method=method, sol=sol, native=False, block=1024)
    key = lambda tr: [(r.t, r.m, r.k, r.event, r.delta_tilde, r.delta_exact) for r in tr.records]  # noqa: E731
    assert key(t1) == key(t2)
    assert np.array_equal(x1, x2)


# ------------------------------------------------------------ plain CG / tri_solve
def _np_cg(A, B, nu, lam, x0, T, tol=0.0):
    """The reference CG recursion (solvers.py:104-140) restated in numpy."""
    Hm = lambda X: A.T @ (A @ X) + nu**2 * lam[:, None] * X  # noqa: E731  (problem.py:89-95)
    x = x0[:, None].copy()
    r = B[:, None] - Hm(x)
    q = r.copy()
    rs = np.sum(r * r, axis=0)
    dts = [0.5 * rs.sum()]
    for _ in range(T):
        active = rs > 0.0
        if not active.any() or 0.5 * rs.sum() <= tol:
            break
        Hq = Hm(q)
        qHq = np.sum(q * Hq, axis=0)
        alpha = np.where(active, rs / np.where(qHq > 0, qHq, 1.0), 0.0)
        x += q * alpha
        r -= Hq * alpha
        rs_new = np.sum(r * r, axis=0)
        q = r + q * np.where(active, rs_new / np.where(rs > 0, rs, 1.0), 0.0)
        rs = rs_new
        dts.append(0.5 * rs.sum())
    return x[:, 0], np.array(dts)


def test_plain_cg_matches_reference_recursion():
    import paper_2104_14101_b200 as ak

    # well conditioned (CG's late iterates amplify rounding differences on
    # ill-conditioned systems, so compare where the recursion is stable)
    rng = np.random.default_rng(11)
    n, d = 600, 40
    A = rng.standard_normal((n, d)) / np.sqrt(n) * (0.98 ** np.arange(d))
    b = rng.standard_normal(d)
    lam = rng.uniform(1, 3, d)
    p = ak.RegularizedProblem(A, b, 0.3, lam)
    x, tr = ak.cg(p, np.zeros(d), 12)
    xr, dts = _np_cg(A, b, 0.3, lam, np.zeros(d), 12)
    got = np.array([r.delta_tilde for r in tr.records])
    assert len(got) == len(dts)
    # late iterations sit at the rounding floor: compare relative to delta_0
    np.testing.assert_allclose(got, dts, rtol=1e-6, atol=1e-12 * dts[0])
    np.testing.assert_allclose(x, xr, rtol=1e-8, atol=1e-10)
    # tol stop
    _, tr2 = ak.cg(p, np.zeros(d), 12, tol=dts[5] * (1 + 1e-6))
    assert len(tr2.records) == 6


@pytest.mark.parametrize("k,c,transposed", [(1, 1, False), (37, 1, False), (37, 3, True), (300, 2, False),
                                            (300, 1, True)])
def test_tri_solve_matches_scipy(k, c, transposed):
    import scipy.linalg

    import paper_2104_14101_b200 as ak

    rng = np.random.default_rng(k + c)
    L = np.tril(rng.standard_normal((k, k))) + 3 * np.eye(k)
    z = rng.standard_normal((k, c)) if c > 1 else rng.standard_normal(k)
    got = ak.tri_solve(L, z, transposed=transposed)
    ref = scipy.linalg.solve_triangular(L, z, lower=True, trans=1 if transposed else 0)
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-12)
    with pytest.raises(ak.DimensionMismatch):
        ak.tri_solve(L, np.ones(k + 1))


# ------------------------------------------------------------ incremental sketch growth
@pytest.mark.parametrize("family,method,dtype", [("srht", "pcg", "float64"), ("gaussian", "ihs", "float64"),
                                                 ("srht-block", "pcg", "float64"), ("gaussian", "ihs", "float32")])
def test_incremental_growth_matches_oracle(family, method, dtype):
    import paper_2104_14101_b200 as ak

    rng = np.random.default_rng(4)
    n, d = 3000, 60
    A = rng.standard_normal((n, d)) / np.sqrt(n) * (0.9 ** np.arange(d))
    b = A.T @ (A @ rng.standard_normal(d) + 0.01 * rng.standard_normal(n))
    nu, T, seed, m0 = 0.05, 8, 3, 4
    block = 1024
    A_used = A.astype(np.float32).astype(np.float64) if dtype == "float32" else A
    p = ak.RegularizedProblem(A, b, nu, dtype=dtype)
    cfg = ak.AdaptiveConfig.for_method(method, 0.125, m0, T, family, seed)
    x, tr = ak.adaptive_run(p, np.zeros(d), cfg, method=method, incremental=True, block=block)
    po = O.Problem.make(A_used, b, nu, np.ones(d))
    sk = O.IncrementalSketcher(family, seed, block=block)
    cap = O.padded_rows(n) if family == "srht" else (min(n, O.padded_rows(block)) if family == "srht-block" else n)
    xo, tro = O.adaptive_run(po, np.zeros(d), method, 0.125, m0, T, "srht" if family != "gaussian" else family,
                             seed, sketcher=sk, cap=cap)
    assert tr.schedule() == tro.schedule()
    tol = 1e-4 if dtype == "float32" else 1e-8
    assert np.linalg.norm(x - xo[:, 0]) <= tol * np.linalg.norm(xo)
    # growth: no redraws -- every resketch keeps the sketch-0 seed, and m doubles
    ms = [m for _, m in tr.schedule()]
    assert ms == sorted(ms)


def test_incremental_tf32_gaussian_converges():
    """TF32 sketches perturb the decrements at the 1e-3 level, so the decision
    times may differ from the fp64 oracle; the solve must still reach the
    fp32 target and grow (not redraw) its sketch."""
    import paper_2104_14101_b200 as ak

    rng = np.random.default_rng(6)
    n, d = 4096, 64
    A = (rng.standard_normal((n, d)) / np.sqrt(n) * (1.0 / np.arange(1, d + 1))).astype(np.float32)
    b = A.astype(np.float64).T @ (A.astype(np.float64) @ rng.standard_normal(d))
    p = ak.RegularizedProblem(A, b, 0.01, dtype="float32")
    sol = ak.direct_solve(p)
    cfg = ak.AdaptiveConfig.for_method("ihs", 0.125, 8, 12, "gaussian", 1)
    x, tr = ak.adaptive_run(p, np.zeros(d), cfg, method="ihs", incremental=True, tf32=True, sol=sol)
    d0 = tr.records[0].delta_exact
    assert tr.records[-1].delta_exact <= 1e-6 * d0
    ms = [m for _, m in tr.schedule()]
    assert ms == sorted(ms) and all(b == 2 * a for a, b in zip([8] + ms[:-1], ms))


@pytest.mark.parametrize("method", ["pcg", "ihs"])
def test_native_driver_reports_not_positive_definite(method):
    """The native driver reads the Cholesky pivot check after the restart's
    synchronization (no sync of its own); a non-finite sketch still raises
    NotPositiveDefinite, as the reference's build does (preconditioner.py:60-74)."""
    import paper_2104_14101_b200 as ak
    from paper_2104_14101_b200.errors import NotPositiveDefinite

    rng = np.random.default_rng(5)
    A = rng.standard_normal((2048, 40))
    A[77, 3] = np.nan
    b = rng.standard_normal(40)
    p = ak.RegularizedProblem(A, b, 1e-1, None, validate=False)
    cfg = ak.AdaptiveConfig.for_method(method, 0.125, 8, 4, "sjlt", 1)
    with pytest.raises(NotPositiveDefinite):
        ak.adaptive_run(p, np.zeros(40), cfg, method=method, native=True)
