"""Multi-rank host logic on CPU (gloo, world_size 2): row-shard plan, the
global-index randomness of the sharded sketches and the all-reduce exchange
steps, with the oracle as the per-shard compute.  The GPU path uses the same
ShardPlan / Comm / index conventions (paper_2104_14101_b200/parallel.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import adasketch_oracle as O
from paper_2104_14101_b200.parallel import Comm, shard_rows


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm()
        rng = np.random.default_rng(0)
        n, d, m, seed, nu = 1003, 7, 13, 42, 0.3
        A = rng.standard_normal((n, d))
        lam = 1.0 + rng.uniform(0, 2, d)
        x = rng.standard_normal(d)
        plan = shard_rows(n, world, rank)
        Al = A[plan.row0:plan.row0 + plan.n_local]
        # SJLT (non power-of-two m: rejection-aware global draw indices)
        sa = torch.from_numpy(O.sjlt_shard(Al, m, seed, plan.row0, n))
        comm.all_reduce_sum_(sa)
        full = O.sketch_sjlt(A, m, seed)
        # Gaussian: Philox columns keyed by global row index
        sg = torch.from_numpy(O.philox_gaussian(m, plan.n_local, seed, col0=plan.row0) @ Al)
        comm.all_reduce_sum_(sg)
        fullg = O.sketch_gaussian(A, m, seed)
        # block-SRHT with block-aligned shards
        block = 256
        pb = shard_rows(n, world, rank, align=block)
        Ab = A[pb.row0:pb.row0 + pb.n_local]
        sb = np.zeros((m, d))
        for r0 in range(0, pb.n_local, block):
            bidx = (pb.row0 + r0) // block
            sb += O.sketch_srht(Ab[r0:r0 + block], m, O.derive_seed(seed, bidx))
        sb = torch.from_numpy(sb)
        comm.all_reduce_sum_(sb)
        fullb = O.block_srht(A, m, seed, block)
        # partial A^T A x + regularizer after the all-reduce
        hp = torch.from_numpy(Al.T @ (Al @ x))
        comm.all_reduce_sum_(hp)
        hx = hp.numpy() + nu**2 * lam * x
        fullh = O.Problem.make(A, np.zeros(d), nu, lam).hess_mult(x)
        q.put((rank, np.abs(sa.numpy() - full).max(), np.abs(sg.numpy() - fullg).max(),
               np.abs(sb.numpy() - fullb).max(), np.abs(hx - fullh).max() / np.abs(fullh).max()))
    finally:
        dist.destroy_process_group()


def test_sharded_exchanges_match_unsharded_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e_sjlt, e_gauss, e_bsrht, e_hess in res:
        assert e_sjlt < 1e-12 and e_gauss < 1e-12 and e_bsrht < 1e-12 and e_hess < 1e-13


@pytest.mark.parametrize("n,world,align", [(1003, 2, 1), (1 << 20, 8, 1 << 17), (10, 4, 1), (5, 8, 1)])
def test_shard_plan_covers_rows(n, world, align):
    plans = [shard_rows(n, world, r, align) for r in range(world)]
    assert plans[0].row0 == 0
    for a, b in zip(plans, plans[1:]):
        assert a.row0 + a.n_local == b.row0
        assert b.row0 % align == 0 or b.row0 == n
    assert plans[-1].row0 + plans[-1].n_local == n
