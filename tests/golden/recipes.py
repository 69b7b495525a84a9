"""Deterministic inputs shared by make_golden.py and the tests (so the
fixture stores only outputs, not inputs)."""
import numpy as np

SRHT_CASES = [(64, 3, 64, 4), (300, 4, 128, 1), (1000, 7, 500, 2), (5000, 17, 3000, 6), (1, 2, 1, 0),
              (4096, 9, 32, 11), (20001, 3, 400, 5)]
SJLT_CASES = [(64, 5, 16, 9), (1000, 37, 64, 3), (5000, 13, 1000, 4), (20, 8, 1, 2), (333, 16, 333, 8),
              (4097, 6, 3, 7)]
SJLT_S_CASES = [(200, 6, 16, 25, 3), (50, 4, 7, 3, 2)]
FWHT_CASES = [(1, 1), (8, 3), (256, 5), (4096, 2)]
DERIVE = [(0, 0), (1, 0), (1, 1), (1, 7), (7, 31), (2**40 + 3, 2), (123456789, 1000)]
PRE_CASES = [(40, 10), (10, 10), (6, 10), (300, 200), (100, 300)]
# (method, family, n, d, decay (None -> j^-0.5), nu, lam uniform, m_init, T)
RUNS = [("pcg", "srht", 4096, 128, 0.98, 1e-2, False, 8, 8),
        ("pcg", "sjlt", 8192, 128, None, 1e-3, True, 8, 8),
        ("ihs", "gaussian", 2048, 64, None, 1e-1, False, 4, 8),
        ("ihs", "srht", 1000, 32, 0.9, 5e-2, False, 2, 6)]


def sketch_input(kind: str, i: int, n: int, d: int) -> np.ndarray:
    base = {"srht": 1000, "sjlt": 2000, "sjlts": 3000, "fwht": 4000}[kind]
    return np.random.default_rng(base + i).standard_normal((n, d))


def pre_inputs():
    rng = np.random.default_rng(5000)
    out = []
    for m, d in PRE_CASES:
        SA = rng.standard_normal((m, d))
        lam = 1.0 + rng.uniform(0, 2, d)
        Z = rng.standard_normal((d, 3))
        out.append((SA, lam, Z))
    A = rng.standard_normal((500, 40))
    B = rng.standard_normal((40, 2))
    lam = 1.0 + rng.uniform(0, 2, 40)
    X = rng.standard_normal((40, 2))
    return out, (A, B, lam, X)


def run_instance(i: int):
    method, fam, n, d, decay, nu, lam_u, m0, T = RUNS[i]
    r = np.random.default_rng(6000 + i)
    G = r.standard_normal((n, d)) / np.sqrt(n)
    V, _ = np.linalg.qr(r.standard_normal((d, d)))
    j = np.arange(1, d + 1, dtype=float)
    sig = decay**j if decay else j**-0.5
    A = (G * sig[None, :]) @ V.T
    b = A.T @ (A @ r.standard_normal(d) + 0.01 * r.standard_normal(n))
    lam = np.random.default_rng(123).uniform(1, 10, d) if lam_u else np.ones(d)
    return A, b, lam
