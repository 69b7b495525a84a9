"""Row-sharded data parallelism over A (one process per GPU).

The reference is single-process (SPEC.md:8, :485 list distributed execution
as a non-goal); this is the B200 build's extension for configs 2-4.  A is
split into contiguous row shards; d-vectors, the sketch SA and the
preconditioner factor are replicated.  Exchanges:

* every loop pass: one all-reduce of the d*c partial A_g^T (A_g x), issued
  from inside the fused C-ABI iteration body through its allreduce hook, so
  the single-GPU and sharded solvers run the same code;
* every resketch: one all-reduce of the m x d partial sketch S_g A_g.

Randomness is indexed globally, so the sketch does not depend on the shard
count (up to the order of the cross-shard sum):
* SJLT: bucket / sign of global row i = draws i and n_total + i of the
  reference's PCG64 stream (libadask jump-ahead, row0 / n_total arguments);
* Gaussian: Philox counter = (sketch row, global A row);
* block-SRHT: fixed-size row blocks (independent of the shard count), block b
  sketched with derive_seed(seed, b), blocks summed.  The global SRHT does
  not shard (its butterflies cross every row), so it runs replicated.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from . import device as dv
from .embeddings import SketchSpec, derive_seed, gaussian_dev, sjlt_dev, srht_dev
from .problem import RegularizedProblem

__all__ = ["ShardPlan", "shard_rows", "Comm", "ShardedProblem", "sharded_sketcher", "block_srht_sketcher"]


@dataclass(frozen=True)
class ShardPlan:
    n_total: int
    world: int
    rank: int
    row0: int
    n_local: int


def shard_rows(n_total: int, world: int, rank: int, align: int = 1) -> ShardPlan:
    """Contiguous balanced row shards; boundaries on multiples of `align`
    (the block-SRHT block size) so that no block straddles two ranks."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    units = -(-n_total // align)
    u0 = units * rank // world
    u1 = units * (rank + 1) // world
    row0 = min(u0 * align, n_total)
    row1 = min(u1 * align, n_total)
    return ShardPlan(n_total, world, rank, row0, row1 - row0)


class Comm:
    """The shard group.  torch.distributed is the plumbing (rendezvous,
    the NCCL unique-id broadcast, gloo in the CPU tests); with the NCCL
    backend on GPUs, libadask gets its own NCCL communicator on this rank's
    device (adask_comm_init_nccl) and the native solve issues every exchange
    itself on its stream (`native`).  all_reduce_sum_ serves the Python-level
    paths (custom sketchers, ShardedProblem.hess_mult_dev)."""

    def __init__(self, group=None, *, native: bool | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        backend = dist.get_backend(group)
        if native is None:
            native = backend == "nccl" and torch.cuda.is_available()
        self.native = False
        if native:
            self._init_native()

    def _init_native(self) -> None:
        lib = _lib.lib()
        if not lib.adask_nccl_available():
            raise RuntimeError("libadask could not load libnccl.so.2 for the native shard communicator")
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            _lib.check(lib.adask_nccl_unique_id(uid), "nccl_unique_id")
        obj = [bytes(uid)]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        C.memmove(uid, obj[0], 128)
        _lib.check(lib.adask_comm_init_nccl(dv.ctx().handle, uid, self.rank, self.world), "comm_init_nccl")
        self.native = True

    def all_reduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t


class _CudaView:
    """__cuda_array_interface__ wrapper so a raw device pointer handed to the
    allreduce hook becomes a torch tensor without a copy."""

    def __init__(self, ptr: int, count: int, dtype: int = _lib.F64):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8" if dtype == _lib.F64 else "<f4",
                                         "data": (ptr, False), "version": 3, "strides": None}


class ShardedProblem(RegularizedProblem):
    """RegularizedProblem over this rank's rows [row0, row0 + n_local) of a
    row-sharded A; H X all-reduces the partial A_local^T A_local X."""

    def __init__(self, A_local, B, nu, lam=None, *, plan: ShardPlan, comm: Comm, **kw):
        super().__init__(A_local, B, nu, lam, row0=plan.row0, n_total=plan.n_total, **kw)
        self.plan = plan
        self.comm = comm

        def _hook(ptr, count, dtype, user, stream):
            try:
                t = torch.as_tensor(_CudaView(int(ptr), int(count), int(dtype)), device=self.A_dev.device)
                self.comm.all_reduce_sum_(t)
                return 0
            except Exception:  # reported through the C status path
                return 1

        self._hook = _lib.ALLREDUCE_FN(_hook)  # keep alive

    def descriptor(self) -> _lib.Problem:
        pb = super().descriptor()
        if self.comm.native:
            pb.use_ctx_comm = 1  # exchanges on libadask's NCCL communicator
        else:
            pb.allreduce = self._hook  # host hook (gloo)
            pb.allreduce_user = None
        pb.comm_rank = self.comm.rank
        pb.comm_world = self.comm.world
        return pb

    def hess_mult_dev(self, Xt, out=None, *, minus_B=False, partial=False):
        part = super().hess_mult_dev(Xt, out, minus_B=False, partial=True)
        if partial:
            return part
        self.comm.all_reduce_sum_(part)
        c, d = part.shape
        B = self.Bt if minus_B else None
        _lib.check(_lib.lib().adask_vec_hess_finish(dv.ctx().handle, part.data_ptr(), d, c, d,
                                                    Xt.contiguous().data_ptr(), self.nu**2,
                                                    self.lam_dev.data_ptr(),
                                                    None if B is None else B.data_ptr(), part.data_ptr(),
                                                    dv.stream()), "hess_finish")
        return part


def sharded_sketcher(comm: Comm, *, block: int = 1 << 21, tf32: bool = False):
    """sketcher(p, spec) for adaptive_run on a ShardedProblem: local partial
    sketch with global randomness, then all-reduce."""

    def sk(p: RegularizedProblem, spec: SketchSpec) -> torch.Tensor:
        A = p.A_dev
        if spec.family == "sjlt":
            SA = sjlt_dev(A, spec.m, spec.seed, spec.s, row0=p.row0, n_total=p.n_total)
        elif spec.family == "gaussian":
            SA = gaussian_dev(A, spec.m, spec.seed, row0=p.row0, tf32=tf32)
        elif spec.family in ("srht-block", "srht_block"):
            SA = _block_srht_local(A, spec.m, spec.seed, p.row0, block)
        elif spec.family == "srht":
            raise NotImplementedError("the global SRHT does not shard; use family 'srht-block'")
        else:
            raise ValueError(f"unknown sketch family {spec.family!r}")
        return comm.all_reduce_sum_(SA)

    return sk


def _block_srht_local(A: torch.Tensor, m: int, seed: int, row0: int, block: int) -> torch.Tensor:
    n, d = A.shape
    if row0 % block:
        raise ValueError("shard must start on a block boundary")
    SA = torch.zeros((int(m), d), dtype=A.dtype, device=A.device)
    for r0 in range(0, n, block):
        b = (row0 + r0) // block
        srht_dev(A[r0:r0 + block], m, derive_seed(seed, b), out=SA, accumulate=True)
    return SA


def block_srht_sketcher(block: int = 1 << 21):
    """Config 4's block-SRHT on one GPU: SA = sum_b sketch_srht(A_b, m,
    derive_seed(seed, b)) over fixed row blocks, summed in block order."""

    def sk(p: RegularizedProblem, spec: SketchSpec) -> torch.Tensor:
        return _block_srht_local(p.A_dev, spec.m, spec.seed, p.row0, block)

    return sk
