"""Row-sharded native solves on the GPU.

* NCCL world 1 inside libadask (adask_comm_init_nccl): the native driver's
  sharded code -- one all-reduce of the 2d partial pair per PCG proposal,
  reduce-scatter of S_g A_g + partial Gram + d x d all-reduce per dense build,
  SA all-reduce on the Woodbury path -- against the unsharded solve.
* Two ranks on the one GPU over gloo (the host all-reduce hook; no kernel
  waits on another rank): each rank holds half of A (or, for the block SRHT,
  one rank holds every block and the other an EMPTY shard); same schedule and
  x <= 1e-10 as the unsharded solve on rank 0.
The reference is single-process: the oracle here is the
unsharded solve, itself pinned to the reference by the golden tests."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance(n, d, decay, nu, lam_u, seed=0):
    from oracle import adasketch_oracle as O

    j = np.arange(1, d + 1, dtype=float)
    sig = decay**j if decay else j**-0.5
    return O.make_config_problem(n, d, sig, nu, lam_u, data_seed=seed)


def _events(tr):
    return [(r.t, r.m, r.k, r.event) for r in tr.records]


# (method, family, n, d, decay, nu, lam_uniform, m_init, T, block)
CASES = [("pcg", "sjlt", 1 << 14, 128, None, 1e-3, True, 8, 10, 0),
         ("ihs", "gaussian", 1 << 13, 96, 0.95, 1e-2, False, 8, 8, 0),
         ("pcg", "srht-block", 1 << 14, 64, 0.97, 1e-3, True, 8, 8, 1 << 12)]


def test_native_nccl_world1_matches_unsharded():
    import torch.distributed as dist

    import paper_2104_14101_b200 as ak
    from paper_2104_14101_b200.parallel import Comm, ShardedProblem, shard_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        comm = Comm()
        assert comm.native  # libadask owns an NCCL communicator on this device
        for method, fam, n, d, decay, nu, lam_u, m0, T, block in CASES:
            A, b, lam = _instance(n, d, decay, nu, lam_u)
            plan = shard_rows(n, 1, 0, align=block or 1)
            ps = ShardedProblem(A, b, nu, lam, plan=plan, comm=comm)
            p = ak.RegularizedProblem(A, b, nu, lam)
            cfg = ak.AdaptiveConfig.for_method(method, 0.125, m0, T, fam, 1)
            kw = {"block": block} if block else {}
            xs, trs = ak.adaptive_run(ps, np.zeros(d), cfg, method=method, native=True, **kw)
            x1, tr1 = ak.adaptive_run(p, np.zeros(d), cfg, method=method, native=True, **kw)
            assert _events(trs) == _events(tr1), (fam, _events(trs), _events(tr1))
            assert max(r.m for r in tr1.records) >= d  # the dense (reduce-scatter) build ran
            assert np.linalg.norm(xs - x1) <= 1e-10 * np.linalg.norm(x1)
    finally:
        dist.destroy_process_group()


def _rank_worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_14101_b200 as ak
        from paper_2104_14101_b200.parallel import Comm, ShardedProblem, ShardPlan, shard_rows

        method, fam, n, d, decay, nu, lam_u, m0, T, block, empty = case
        A, b, lam = _instance(n, d, decay, nu, lam_u)
        comm = Comm(native=False)  # host all-reduce hook over gloo
        align = block or 1
        if empty:
            # rank 0 holds every block, rank 1 an empty shard (the
            # collectives must pair up whatever the local row count)
            plan = ShardPlan(n, world, rank, 0 if rank == 0 else n, n if rank == 0 else 0)
        else:
            plan = shard_rows(n, world, rank, align)
        Al = np.ascontiguousarray(A[plan.row0:plan.row0 + plan.n_local])
        ps = ShardedProblem(Al, b, nu, lam, plan=plan, comm=comm)
        cfg = ak.AdaptiveConfig.for_method(method, 0.125, m0, T, fam, 1)
        kw = {"block": block} if block else {}
        xs, trs = ak.adaptive_run(ps, np.zeros(d), cfg, method=method, native=True, **kw)
        out = {"rank": rank, "events": _events(trs), "x": xs}
        if rank == 0:
            p = ak.RegularizedProblem(A, b, nu, lam)
            x1, tr1 = ak.adaptive_run(p, np.zeros(d), cfg, method=method, native=True, **kw)
            out.update(events1=_events(tr1), x1=x1)
        q.put(out)
    except Exception as e:  # surfaced by the parent
        q.put({"rank": rank, "error": repr(e)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ci,empty", [(0, False), (1, False), (2, False), (2, True)])
def test_two_ranks_one_gpu_gloo_match_unsharded(ci, empty):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    case = CASES[ci] + (empty,)
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        o = q.get(timeout=300)
        res[o["rank"]] = o
    for p in procs:
        p.join(timeout=120)
    for o in res.values():
        assert "error" not in o, o.get("error")
    r0, r1 = res[0], res[1]
    assert r0["events"] == r1["events"] == r0["events1"]
    assert np.linalg.norm(r0["x"] - r0["x1"]) <= 1e-10 * np.linalg.norm(r0["x1"])
    assert np.array_equal(r0["x"], r1["x"])  # replicated iterate
