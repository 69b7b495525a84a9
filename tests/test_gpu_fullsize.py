"""Parity at BASELINE.json's full sizes through size-independent properties.

The CPU oracle cannot run configs 1-4 at full size in a test, so these
checks use properties that hold at any size:

* column separability: the SRHT, block-SRHT and SJLT act on every column of
  A independently, so the first few columns of the full-size device sketch
  must equal the oracle's sketch of just those columns (bit for bit in fp64);
* the TF32 Gaussian sketch is compared column-wise with the library's fp64
  Philox path (same S definition, checked against the oracle at small sizes);
* H = A^T A + nu^2 Lam is symmetric and linear: x^T (H y) = y^T (H x), and
  H (a x + b y) = a H x + b H y, checked on the one-pass kernel at full size;
* the two-column proposal pass equals two single-column passes bitwise;
* configs 1-2 end to end: native driver == reference-faithful Python loop
  (bitwise traces and x), and x reaches the config's target error.
"""
import numpy as np
import pytest
import torch

from oracle import adasketch_oracle as O

pytestmark = pytest.mark.gpu

COLS = 4  # leading columns compared against the oracle


@pytest.fixture(scope="module")
def ak():
    import paper_2104_14101_b200 as ak

    return ak


def _instance(index, n=None):
    from paper_2104_14101_b200 import configs

    cfg = configs.CONFIGS[index]
    A, _, _ = configs.make_instance_device(cfg, n=n)
    return cfg, A


def test_srht_full_config1_columns_bitwise(ak):
    """Config 1 (2^16 x 1024 fp64), the largest sketch of its schedule."""
    from paper_2104_14101_b200.embeddings import srht_dev

    cfg, A = _instance(1)
    for m in (32, 4096):
        SA = srht_dev(A, m, 7)
        ref = O.sketch_srht(A[:, :COLS].cpu().numpy(), m, 7)
        assert np.array_equal(SA[:, :COLS].cpu().numpy(), ref), m
    del A


def test_block_srht_full_config4_block_columns(ak):
    """Config 4's block SRHT on one full 2^21-row fp32 block, m = 32768
    (the 10-bit pass 2 per half plus combine): the first columns against the
    fp64 oracle within fp32 rounding."""
    from paper_2104_14101_b200.embeddings import srht_dev

    cfg, A = _instance(4, n=1 << 21)
    m = 32768
    SA = srht_dev(A, m, 11)
    ref = O.sketch_srht(A[:, :COLS].double().cpu().numpy(), m, 11)
    got = SA[:, :COLS].double().cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref)
    del A, SA


def test_sjlt_full_config2_columns_bitwise(ak):
    """Config 2 (2^20 x 2048 fp64), the largest sketch of its schedule (m = 65536)."""
    from paper_2104_14101_b200.embeddings import sjlt_dev

    cfg, A = _instance(2)
    for m in (64, 65536):
        SA = sjlt_dev(A, m, 5)
        ref = O.sketch_sjlt(A[:, :COLS].cpu().numpy(), m, 5)
        assert np.array_equal(SA[:, :COLS].cpu().numpy(), ref), m
    del A


def test_gaussian_tf32_full_config3_columns(ak):
    """Config 3 (2^21 x 4096 fp32, m = 2048) on tcgen05 vs the fp64 Philox path
    on the first columns: within the TF32 operand rounding."""
    from paper_2104_14101_b200.embeddings import gaussian_dev

    cfg, A = _instance(3)
    m = 2048
    SA = gaussian_dev(A, m, 3, tf32=True)
    ref = gaussian_dev(A[:, :COLS].double().contiguous(), m, 3)
    got = SA[:, :COLS].double()
    assert float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref)) <= 2e-3
    del A, SA


@pytest.mark.parametrize("index", [2, 4])
def test_hess_mult_full_symmetry_linearity(ak, index):
    """The one-pass A^T (A x) kernel at configs 2 (16 GiB fp64) and 4 (64 GiB
    fp32): symmetric and linear to rounding."""
    cfg, A = _instance(index)
    d = cfg.d
    lam = torch.from_numpy(np.random.default_rng(1).uniform(1, 10, d)).cuda()
    p = ak.RegularizedProblem(A, torch.zeros(d, dtype=torch.float64, device="cuda"), cfg.nu, lam,
                              validate=False)
    g = torch.Generator(device="cuda").manual_seed(index)
    X = torch.randn(2, d, dtype=torch.float64, device="cuda", generator=g)
    HX = p.hess_mult_dev(X)
    x, y = X[0], X[1]
    Hx, Hy = HX[0], HX[1]
    sym = float(torch.dot(x, Hy) - torch.dot(y, Hx)) / float(torch.dot(x, Hx).abs())
    tol = 1e-12 if cfg.dtype == "float64" else 1e-5
    assert abs(sym) <= tol
    Z = (2.5 * x - 0.75 * y)[None, :]
    HZ = p.hess_mult_dev(Z)[0]
    lin = torch.linalg.norm(HZ - (2.5 * Hx - 0.75 * Hy)) / torch.linalg.norm(HZ)
    assert float(lin) <= tol
    del A, p


def test_pair_pass_equals_single_passes_full_config1(ak):
    """The two-column proposal pass (restart reuse) against two single-column
    passes at config 1: bitwise."""
    from paper_2104_14101_b200 import _lib
    from paper_2104_14101_b200 import device as dv

    cfg, A = _instance(1)
    d = cfg.d
    lam = torch.ones(d, dtype=torch.float64, device="cuda")
    B = torch.randn(d, dtype=torch.float64, device="cuda")
    p = ak.RegularizedProblem(A, B, cfg.nu, lam, validate=False)
    g = torch.Generator(device="cuda").manual_seed(9)
    X = torch.randn(2, d, dtype=torch.float64, device="cuda", generator=g)
    single = p.hess_mult_dev(X)  # column by column
    fused = torch.empty_like(X)
    status = _lib.lib().adask_hess_mult_pair(dv.ctx().handle, dv.dtype_code(A.dtype), A.data_ptr(), A.shape[0], d,
                                              A.stride(0), X[0].data_ptr(), X[1].data_ptr(), cfg.nu ** 2,
                                              lam.data_ptr(), fused[0].data_ptr(), fused[1].data_ptr(),
                                              dv.stream())
    _lib.check(status, "hess_mult_pair")
    assert torch.equal(single, fused)
    del A, p


@pytest.mark.parametrize("index", [1, 2])
def test_adaptive_full_native_equals_python_loop(ak, index):
    """Configs 1 and 2 at full size: the native driver (restart reuse, fused
    bodies) and the reference-faithful Python loop give bitwise-identical
    traces and x, and x reaches the config's target relative error."""
    from paper_2104_14101_b200 import configs

    cfg = configs.CONFIGS[index]
    A, b, lam = configs.make_instance_device(cfg)
    p = ak.RegularizedProblem(A, b, cfg.nu, lam, validate=False)
    sol = ak.direct_solve(p)
    acfg = ak.AdaptiveConfig.for_method(cfg.method, 0.125, cfg.m_init, cfg.t_star, cfg.family, 1)
    x0 = torch.zeros(cfg.d, dtype=torch.float64, device="cuda")
    x1, t1 = ak.adaptive_run(p, x0, acfg, method=cfg.method, sol=sol, native=True)
    x2, t2 = ak.adaptive_run(p, x0, acfg, method=cfg.method, sol=sol, native=False)
    key = lambda tr: [(r.t, r.m, r.k, r.event, r.delta_tilde, r.delta_exact) for r in tr.records]  # noqa: E731
    assert key(t1) == key(t2)
    assert torch.equal(x1, x2)
    d0 = t1.records[0].delta_exact
    assert ak.exact_error(p, x1, sol) <= cfg.target * d0
    del A, p
