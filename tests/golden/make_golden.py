"""Generate tests/golden/reference_golden.npz from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package `adasketch` from /root/reference/pkg/src
(read-only) and records its outputs on small seeded inputs: derive_seed
values, SRHT / SJLT sketches (and the sign / bucket / row draws in the
reference's draw order), fwht, preconditioner solves on both paths,
hess_mult / gradient, direct_solve, and full adaptive_run traces for the
three sketch families.  tests/test_oracle_golden.py pins the CPU oracle
(oracle/adasketch_oracle.py) against this file; tests/test_gpu_golden.py pins
the GPU path.  The fixture is committed; /root/reference is never read at
test time.
"""
from __future__ import annotations

import importlib.util
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src/adasketch/__init__.py"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "adasketch_ref", REF, submodule_search_locations=[os.path.dirname(REF)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["adasketch_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from recipes import (DERIVE, FWHT_CASES, RUNS, SJLT_CASES, SJLT_S_CASES, SRHT_CASES, pre_inputs,  # noqa: E402
                     run_instance, sketch_input)


def main() -> None:
    ref = load_reference()
    g: dict[str, np.ndarray] = {}
    g["derive_in"] = np.array(DERIVE, dtype=np.uint64)
    g["derive_out"] = np.array([ref.derive_seed(b, k) for b, k in DERIVE], dtype=np.uint64)
    for i, (n, d, m, seed) in enumerate(SRHT_CASES):
        A = sketch_input("srht", i, n, d)
        g[f"srht{i}_SA"] = ref.sketch_srht(A, m, seed).SA
        rng = np.random.default_rng(seed)  # the reference's draw order, embeddings.py:95-100
        g[f"srht{i}_bits"] = rng.integers(0, 2, size=n).astype(np.int8)
        g[f"srht{i}_idx"] = rng.choice(ref.padded_rows(n), size=m, replace=False)
        g[f"srht{i}_meta"] = np.array([n, d, m, seed])
    for i, (n, d, m, seed) in enumerate(SJLT_CASES):
        A = sketch_input("sjlt", i, n, d)
        g[f"sjlt{i}_SA"] = ref.sketch_sjlt(A, m, seed).SA
        rng = np.random.default_rng(seed)  # embeddings.py:117-124
        g[f"sjlt{i}_rows"] = rng.integers(0, m, size=n)
        g[f"sjlt{i}_bits"] = rng.integers(0, 2, size=n).astype(np.int8)
        g[f"sjlt{i}_meta"] = np.array([n, d, m, seed])
    for i, (n, d, m, seed, s) in enumerate(SJLT_S_CASES):
        A = sketch_input("sjlts", i, n, d)
        g[f"sjlts{i}_SA"] = ref.sketch_sjlt(A, m, seed, s=s).SA
        g[f"sjlts{i}_meta"] = np.array([n, d, m, seed, s])
    for i, (n, d) in enumerate(FWHT_CASES):
        x = sketch_input("fwht", i, n, d)
        g[f"fwht{i}_y"] = ref.fwht(x)
        g[f"fwht{i}_yu"] = ref.fwht(x, normalized=False)
    # preconditioner both paths
    pres, (A, B, lam, X) = pre_inputs()
    for i, (SA, lamv, Z) in enumerate(pres):
        P = ref.build(SA, 0.7, lamv)
        g[f"pre{i}_out"] = P.solve(Z)
        g[f"pre{i}_L"] = P.L
        g[f"pre{i}_path"] = np.array([0 if P.path == "cholesky-d" else 1])
        g[f"pre{i}_dec"] = np.array([ref.approx_newton_decrement(P, Z)])
    # problem
    p = ref.RegularizedProblem(A=A, B=B, nu=0.8, lam=lam)
    g["prob_HX"] = p.hess_mult(X)
    g["prob_grad"] = p.gradient(X)
    xs = ref.direct_solve(p).x_star
    g["prob_xstar"] = xs
    g["prob_err"] = np.array([ref.exact_error(p, X, ref.ExactSolution(xs))])
    # adaptive runs (reference driver, its own sketches)
    for i, (method, fam, n, d, decay, nu, lam_u, m0, T) in enumerate(RUNS):
        A, b, lam = run_instance(i)
        p = ref.RegularizedProblem(A=A, B=b, nu=nu, lam=lam)
        sol = ref.direct_solve(p)
        cfg = ref.AdaptiveConfig.for_method(method, 0.125, m0, T, fam, 1)
        x, tr = ref.adaptive_run(p, np.zeros(d), cfg, method=method, sol=sol)
        g[f"run{i}_x"] = x
        g[f"run{i}_xstar"] = sol.x_star
        g[f"run{i}_rec"] = np.array([[rec.t, rec.m, rec.k, ["plain", "accepted", "resketch"].index(rec.event),
                                      rec.delta_tilde, rec.delta_exact] for rec in tr.records])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1024:.0f} KiB "
          f"(numpy {np.__version__})")


if __name__ == "__main__":
    main()
