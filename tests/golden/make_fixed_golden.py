"""Fixed-sketch solver fixtures (ihs_run, pcg_run, polyak_ihs_run, cg) from the
REFERENCE implementation (/root/reference/pkg/src/adasketch/solvers.py:104-140,
157-224, 293-328), run in the build container:

    python tests/golden/make_fixed_golden.py

The sketches are SRHT / SJLT, whose draws the device reproduces bit for bit,
so the reference runs on its own code path.  Output:
tests/golden/fixed_golden.npz (traces and iterates).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402
from recipes import FIXED_RUNS, fixed_instance  # noqa: E402


def main() -> None:
    ref = load_reference()
    g = {}
    for i, (solver, fam, n, d, c, m, rho, seed, T, tol, s) in enumerate(FIXED_RUNS):
        A, B, lam, nu = fixed_instance(i)
        p = ref.RegularizedProblem(A=A, B=B, nu=nu, lam=lam)
        sol = ref.direct_solve(p)
        x0 = np.zeros((d, c)) if c > 1 else np.zeros(d)
        if solver == "ihs":
            x, tr = ref.ihs_run(p, x0, m, rho, fam, seed, T, sol=sol, s=s)
        elif solver == "pcg":
            x, tr = ref.pcg_run(p, x0, m, fam, seed, T, tol=tol, sol=sol, s=s)
        elif solver == "polyak":
            x, tr = ref.polyak_ihs_run(p, x0, m, rho, fam, seed, T, sol=sol, s=s)
        else:
            x, tr = ref.cg(p, x0, T, tol=tol, sol=sol)
        g[f"f{i}_x"] = np.asarray(x)
        g[f"f{i}_rec"] = np.array([[r.t, r.m, r.delta_tilde, r.delta_exact] for r in tr.records])
    out = os.path.join(HERE, "fixed_golden.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out}: {len(g)} arrays")


if __name__ == "__main__":
    main()
