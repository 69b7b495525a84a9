"""`adasketch` drop-in shim: the reference package's API with every hot-path
name served by paper_2104_14101_b200 (GPU, libadask).

Used to run the REFERENCE's own test suite against the B200 build
(tools/run_reference_suite.py).  The reference package is loaded from an
untracked working copy (.refsuite/src/adasketch, made by
`tools/run_reference_suite.py --prepare` in the build container; it is
git-ignored and never committed) under the alias `_adasketch_ref`; then the
hot-path names -- the sketches, Cholesky / triangular solve / FWHT, the
preconditioner, the problem's H x and direct solve, every solver and the
error classes -- are replaced in ALL of its modules (so the reference's
out-of-scope helpers, e.g. diagnostics or the CLI, call the GPU code too),
and the patched package is installed as `adasketch`.  The Gaussian sketch
runs in the opt-in rng="numpy" mode (the reference's own ziggurat draw,
applied on the GPU), so seed-pinned tests see the reference's randomness.
"""
import importlib
import importlib.util
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)
_SRC = os.environ.get("ADASK_REF_SRC", os.path.join(_ROOT, ".refsuite", "src", "adasketch"))
if not os.path.exists(os.path.join(_SRC, "__init__.py")):
    raise ImportError(f"reference package not found at {_SRC} (run tools/run_reference_suite.py --prepare)")

_spec = importlib.util.spec_from_file_location("_adasketch_ref", os.path.join(_SRC, "__init__.py"),
                                               submodule_search_locations=[_SRC])
_ref = importlib.util.module_from_spec(_spec)
sys.modules["_adasketch_ref"] = _ref
_spec.loader.exec_module(_ref)
_SUBS = ("errors", "linalg", "embeddings", "problem", "preconditioner", "solvers", "diagnostics", "cli")
for _s in _SUBS:
    importlib.import_module("_adasketch_ref." + _s)

import paper_2104_14101_b200 as _ak  # noqa: E402
from paper_2104_14101_b200 import embeddings as _emb  # noqa: E402
from paper_2104_14101_b200 import errors as _err  # noqa: E402
from paper_2104_14101_b200 import linalg as _lin  # noqa: E402
from paper_2104_14101_b200 import preconditioner as _pre  # noqa: E402
from paper_2104_14101_b200 import problem as _prob  # noqa: E402
from paper_2104_14101_b200 import solvers as _sol  # noqa: E402

_emb.set_gaussian_rng("numpy")

HOT_PATH = {
    # embeddings.py:56-140
    "SketchSpec": _emb.SketchSpec, "SketchedData": _emb.SketchedData, "derive_seed": _emb.derive_seed,
    "padded_rows": _emb.padded_rows, "sketch": _emb.sketch, "sketch_gaussian": _emb.sketch_gaussian,
    "sketch_srht": _emb.sketch_srht, "sketch_sjlt": _emb.sketch_sjlt,
    # linalg.py:30-88
    "cholesky": _lin.cholesky, "tri_solve": _lin.tri_solve, "fwht": _lin.fwht,
    # preconditioner.py:26-88
    "Preconditioner": _pre.Preconditioner, "build": _pre.build,
    "approx_newton_decrement": _pre.approx_newton_decrement,
    # problem.py:41-158
    "RegularizedProblem": _prob.RegularizedProblem, "ExactSolution": _prob.ExactSolution,
    "direct_solve": _prob.direct_solve, "exact_error": _prob.exact_error,
    # solvers.py:51-659
    "TraceRecord": _sol.TraceRecord, "SolverTrace": _sol.SolverTrace, "AdaptiveConfig": _sol.AdaptiveConfig,
    "adaptive_run": _sol.adaptive_run, "ihs_run": _sol.ihs_run, "ihs_step": _sol.ihs_step,
    "pcg_run": _sol.pcg_run, "polyak_ihs_run": _sol.polyak_ihs_run, "cg": _sol.cg,
}
# the error classes the GPU code raises (same names and hierarchy, errors.py)
HOT_PATH.update({n: getattr(_err, n) for n in dir(_err) if isinstance(getattr(_err, n), type)
                 and issubclass(getattr(_err, n), Exception)})

for _m in [_ref] + [sys.modules["_adasketch_ref." + s] for s in _SUBS]:
    for _name, _obj in HOT_PATH.items():
        if hasattr(_m, _name):
            setattr(_m, _name, _obj)
    # tuples of exception classes built at import time (e.g. the CLI's
    # exit-code groups) must hold the classes the GPU code raises
    for _name, _val in list(vars(_m).items()):
        if isinstance(_val, tuple) and _val and all(isinstance(c, type) for c in _val):
            setattr(_m, _name, tuple(HOT_PATH.get(c.__name__, c) for c in _val))

sys.modules["adasketch"] = _ref
for _s in _SUBS:
    sys.modules["adasketch." + _s] = sys.modules["_adasketch_ref." + _s]
