"""BASELINE.json workload configurations and their synthetic instances.

Instance recipe, in this order:
rng = default_rng(data_seed); G = rng.standard_normal((n, d)) / sqrt(n);
V = qr(rng.standard_normal((d, d))).Q; A = G diag(sigma) V^T;
x0 = rng.standard_normal(d); eps = rng.standard_normal(n);
b = A^T (A x0 + 0.01 eps); Lam = I or default_rng(123).uniform(1, 10, d).
sigma_j uses j = 1..d.  The real datasets of the paper are not used (the
configs are synthetic).  `make_instance` builds it on the host with numpy
(exact recipe, used for parity and configs 0-1); `make_instance_device`
builds the same distribution on the GPU from Philox normals (configs 2-4 at
full size, where host generation would take minutes).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    index: int
    method: str       # "ihs" | "pcg"
    family: str       # "gaussian" | "srht" | "sjlt" | "srht-block"
    n: int
    d: int
    decay: str        # sigma_j formula
    nu: float
    lam_uniform: bool
    m_init: int
    target: float     # relative error delta_T / delta_0
    dtype: str        # "float64" | "float32"
    t_star: int       # accepted iterations to target (oracle-tracked run)
    block: int = 0    # block-SRHT block rows

    def sigma(self) -> np.ndarray:
        j = np.arange(1, self.d + 1, dtype=np.float64)
        return {"j^-1": j**-1.0, "0.98^j": 0.98**j, "j^-0.5": j**-0.5, "0.995^j": 0.995**j}[self.decay]

    def name(self) -> str:
        return (f"cfg{self.index}: ada-{self.method.upper()} {self.family} {self.dtype} "
                f"n={self.n} d={self.d} nu={self.nu:g} m_init={self.m_init} target={self.target:g}")


CONFIGS = {
    0: Config(0, "ihs", "gaussian", 4096, 256, "j^-1", 1e-1, False, 16, 1e-10, "float64", 10),
    1: Config(1, "pcg", "srht", 1 << 16, 1024, "0.98^j", 1e-2, False, 32, 1e-10, "float64", 11),
    2: Config(2, "pcg", "sjlt", 1 << 20, 2048, "j^-0.5", 1e-3, True, 64, 1e-10, "float64", 10),
    3: Config(3, "ihs", "gaussian", 1 << 21, 4096, "j^-1", 1e-2, False, 128, 1e-6, "float32", 6),
    4: Config(4, "pcg", "srht-block", 1 << 24, 1024, "0.995^j", 1e-3, True, 64, 1e-6, "float32", 7,
              block=1 << 21),
}


def make_instance(cfg: Config, data_seed: int = 0, n: int | None = None):
    """Host (numpy) instance: returns (A, b, lam) with A in cfg.dtype."""
    n = cfg.n if n is None else n
    d = cfg.d
    rng = np.random.default_rng(data_seed)
    G = rng.standard_normal((n, d))
    G /= np.sqrt(n)
    V, _ = np.linalg.qr(rng.standard_normal((d, d)))
    x0 = rng.standard_normal(d)
    eps = rng.standard_normal(n)
    A = G @ (cfg.sigma()[:, None] * V.T)
    del G
    b = A.T @ (A @ x0 + 0.01 * eps)
    lam = np.random.default_rng(123).uniform(1.0, 10.0, d) if cfg.lam_uniform else np.ones(d)
    if cfg.dtype == "float32":
        A = A.astype(np.float32)
    return A, b, lam


def make_instance_device(cfg: Config, data_seed: int = 0, n: int | None = None, row0: int = 0,
                         n_local: int | None = None):
    """Device instance with the same distribution: G from the library's
    Philox normals (global row index keyed, so shards are consistent), V from
    a seeded host QR, A = G diag(sigma) V^T and b = A^T (A x0 + 0.01 eps)
    assembled on the GPU.  Returns (A_local (device), b (device), lam (device)).
    For a row shard, b needs the all-reduce of the local A^T(.) parts (done
    by the caller)."""
    import torch

    from .embeddings import gaussian_matrix

    n = cfg.n if n is None else n
    n_local = n if n_local is None else n_local
    d = cfg.d
    dt = torch.float64 if cfg.dtype == "float64" else torch.float32
    rng = np.random.default_rng(data_seed)
    V, _ = np.linalg.qr(rng.standard_normal((d, d)))
    x0 = torch.from_numpy(rng.standard_normal(d)).cuda()
    W = torch.from_numpy(cfg.sigma()[:, None] * V.T).cuda()
    A = torch.empty((n_local, d), dtype=dt, device="cuda")
    partial_b = torch.zeros(d, dtype=torch.float64, device="cuda")
    chunk = max(1, min(n_local, (1 << 28) // (8 * d)))
    seed_g = (data_seed << 32) ^ 0x5EED
    seed_e = (data_seed << 32) ^ 0xE5
    for r0 in range(0, n_local, chunk):
        w = min(chunk, n_local - r0)
        # G rows: column block of a 1 x (n*d) Gaussian stream -> reshape
        Gt = gaussian_matrix(d, w, seed_g, col0=row0 + r0)  # d x w, N(0,1)/sqrt(d)
        G = (Gt.t() * (np.sqrt(d) / np.sqrt(n))).contiguous()
        Ac = G @ W
        eps = gaussian_matrix(1, w, seed_e, col0=row0 + r0)[0]
        partial_b += Ac.t() @ (Ac @ x0 + 0.01 * eps)
        A[r0:r0 + w] = Ac.to(dt)
        del G, Ac, Gt
    lam = (np.random.default_rng(123).uniform(1.0, 10.0, d) if cfg.lam_uniform else np.ones(d))
    return A, partial_b, torch.from_numpy(lam).cuda()
