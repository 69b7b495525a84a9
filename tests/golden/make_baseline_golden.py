"""Solve-level parity fixtures at the BASELINE.json configurations, from the
REFERENCE implementation (run in the build container, where /root/reference
exists):

    python tests/golden/make_baseline_golden.py 1 2 3 4

For each config it rebuilds the instance (recipes.baseline_instance), runs
the reference's adaptive_run (/root/reference/pkg/src/adasketch/solvers.py:585-659)
tracked against its own direct_solve for T_MAX accepted steps, reads T* (the
first accepted step with delta_t / delta_0 <= target) off that trace, and
stores the trace prefix up to T*, the iterate x after T* accepted steps, every
proposal's decrement and decision ratio dt_new / (threshold * dt_I), and
fingerprints of A and b.  Configs 1-2 run at full size with the reference's
own sketches (SRHT, SJLT).  Configs 3-4 run at n/16 on float64 of the fp32
matrix the GPU sees, with the product's sketch definitions injected through
the reference's sketch hook: the Philox Gaussian S (oracle
restatement of rng.cuh) for config 3 and, for config 4, the block SRHT
sum_b sketch_srht(A_b, m, derive_seed(seed_K, b)) computed by the
reference's own sketch_srht.  Output: tests/golden/baseline_cfg{c}.npz
(a few KiB each).  Nothing here is read at test time except the .npz.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from make_golden import load_reference  # noqa: E402
from recipes import BASELINE_N, BLOCK4, T_MAX, baseline_instance, fingerprint  # noqa: E402

from paper_2104_14101_b200.configs import CONFIGS  # noqa: E402
from oracle import adasketch_oracle as O  # noqa: E402

EVENTS = ("plain", "accepted", "resketch")


def philox_sketcher(ref):
    def sk(A, spec):
        m, n = spec.m, A.shape[0]
        SA = np.zeros((m, A.shape[1]))
        step = 8192
        for c0 in range(0, n, step):
            w = min(step, n - c0)
            SA += O.philox_gaussian(m, w, spec.seed, col0=c0) @ A[c0:c0 + w]
        return ref.embeddings.SketchedData(SA=SA, spec=spec, n=n)
    return sk


def block_srht_sketcher(ref, block):
    def sk(A, spec):
        SA = None
        for b, r0 in enumerate(range(0, A.shape[0], block)):
            part = ref.sketch_srht(A[r0:r0 + block], spec.m, ref.derive_seed(spec.seed, b)).SA
            SA = part if SA is None else SA + part
        return ref.embeddings.SketchedData(SA=SA, spec=spec, n=A.shape[0])
    return sk


_REF = None


def run(ci: int) -> None:
    global _REF
    if _REF is None:
        _REF = load_reference()
    ref = _REF
    import importlib
    ref.solvers = importlib.import_module("adasketch_ref.solvers")
    ref.embeddings = importlib.import_module("adasketch_ref.embeddings")
    ref.solvers.sketch = ref.embeddings.sketch  # undo a previous config's injection
    cfg = CONFIGS[ci]
    n = BASELINE_N[ci]
    t0 = time.time()
    A, b, lam = baseline_instance(ci, n)
    print(f"cfg{ci}: instance {A.shape} {A.dtype} in {time.time() - t0:.0f}s", flush=True)
    fam = {"srht-block": "srht"}.get(cfg.family, cfg.family)
    if ci == 3:
        ref.solvers.sketch = philox_sketcher(ref)
    elif ci == 4:
        ref.solvers.sketch = block_srht_sketcher(ref, BLOCK4)
    p = ref.RegularizedProblem(A=A, B=b, nu=cfg.nu, lam=lam)
    sol = ref.direct_solve(p)
    print(f"cfg{ci}: direct solve {time.time() - t0:.0f}s", flush=True)
    # capture every proposal's decrement and the iterate after every commit
    st_cls = ref.solvers._PcgState if cfg.method == "pcg" else ref.solvers._IhsState
    props, xs = [], []
    orig_propose, orig_commit = st_cls.propose, st_cls.commit

    def propose(self):
        out = orig_propose(self)
        props.append(out[0])
        return out

    def commit(self, dt, stash):
        orig_commit(self, dt, stash)
        xs.append(np.array(self.x, copy=True))

    st_cls.propose, st_cls.commit = propose, commit
    acfg = ref.AdaptiveConfig.for_method(cfg.method, 0.125, cfg.m_init, T_MAX[ci], fam, 1)
    x, tr = ref.adaptive_run(p, np.zeros(cfg.d), acfg, method=cfg.method, sol=sol)
    st_cls.propose, st_cls.commit = orig_propose, orig_commit
    print(f"cfg{ci}: tracked run {time.time() - t0:.0f}s", flush=True)
    recs = tr.records
    d0 = recs[0].delta_exact
    t_star = next(r.t for r in recs if r.event == "accepted" and r.delta_exact / d0 <= cfg.target)
    # prefix of the trace for a run with T = t_star (the loop stops right after the t_star-th accept)
    cut = next(i for i, r in enumerate(recs) if r.event == "accepted" and r.t == t_star)
    recs = recs[:cut + 1]
    # decision ratios: replay the control flow over the proposals
    ratios, I, dt_I, t = [], 0, recs[0].delta_tilde, 0
    c_ar, phi = acfg.c_alpha_rho, acfg.phi_rho
    for r, dt_new in zip(recs[1:], props):
        thr = c_ar * phi ** (t + 1 - I)
        ratios.append(dt_new / (thr * dt_I) if dt_I > 0 else 0.0)
        if r.event == "resketch":
            I, dt_I = r.t, r.delta_tilde
        else:
            t += 1
    g = {
        "meta": np.array([ci, n, cfg.d, t_star, BLOCK4 if ci == 4 else 0]),
        "rec": np.array([[r.t, r.m, r.k, EVENTS.index(r.event), r.delta_tilde, r.delta_exact] for r in recs]),
        "x": xs[t_star - 1][:, 0],
        "xstar": np.asarray(sol.x_star)[:, 0] if np.asarray(sol.x_star).ndim == 2 else np.asarray(sol.x_star),
        "ratios": np.array(ratios),
        "A_fp": fingerprint(A),
        "b_fp": fingerprint(b),
    }
    out = os.path.join(HERE, f"baseline_cfg{ci}.npz")
    np.savez_compressed(out, **g)
    sched = [(int(r.t), int(r.m)) for r in recs if r.event == "resketch"]
    print(f"cfg{ci}: T*={t_star} schedule {sched} min|log ratio| "
          f"{np.min(np.abs(np.log(np.maximum(g['ratios'], 1e-300)))):.3g} -> {out} "
          f"({time.time() - t0:.0f}s, numpy {np.__version__})", flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["1", "2", "3", "4"]:
        run(int(a))
