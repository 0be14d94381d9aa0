"""Process-group plumbing for row-sharded SpMM on 1/2/4/8 GPUs.

One process per GPU (torchrun; RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* from
the environment).  The SpMM itself needs no collective: every rank holds an
nnz-balanced row shard of A (``partition.plan_shards``), a replica of B and
its own row slab of C.  The collectives here are set-up and optional
epilogue:

* ``broadcast_dense``  -- replicate B from one rank (NCCL over NVLink on
  the GPU box, gloo on CPU);
* ``gather_rows``      -- collect the unequal C row slabs on a root with
  point-to-point send/recv (``ncclSend``/``ncclRecv`` underneath);
* ``max_over_ranks``   -- the timing reduction the bench contract asks for.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from .partition import ShardPlan, plan_shards, shard_csr

__all__ = ["DistContext", "init_from_env", "broadcast_dense", "gather_rows", "max_over_ranks",
           "local_shard"]


@dataclass(frozen=True)
class DistContext:
    rank: int
    world: int
    local_rank: int
    device: torch.device

    @property
    def is_root(self) -> bool:
        return self.rank == 0


def init_from_env(backend: str | None = None) -> DistContext:
    """Initialise the default process group from the torchrun environment
    (no-op for a single process)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    use_cuda = torch.cuda.is_available()
    device = torch.device("cuda", local) if use_cuda else torch.device("cpu")
    if use_cuda:
        torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        backend = backend or ("nccl" if use_cuda else "gloo")
        kw = {"device_id": device} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
    return DistContext(rank, world, local, device)


def broadcast_dense(t: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """In-place broadcast of a dense operand (B) from ``src``."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(t, src=src, group=group)
    return t


def gather_rows(local: torch.Tensor, plan: ShardPlan, *, root: int = 0, group=None):
    """Gather row-disjoint C slabs (shard g holds rows plan.rows(g)) into the
    full [M, N] matrix on ``root``; other ranks return None."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return local
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if plan.k != world:
        raise ValueError(f"plan has {plan.k} shards for a world of {world}")
    lo, hi = plan.rows(rank)
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} rows, plan says {hi - lo}")
    if rank != root:
        if local.numel():
            dist.send(local.contiguous(), dst=root, group=group)
        return None
    full = torch.empty((int(plan.starts[-1]),) + tuple(local.shape[1:]), dtype=local.dtype,
                       device=local.device)
    full[lo:hi] = local
    reqs = []
    for g in range(world):
        if g == root:
            continue
        a, b = plan.rows(g)
        if b > a:
            reqs.append(dist.irecv(full[a:b], src=g, group=group))
    for r in reqs:
        r.wait()
    return full


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar (e.g. a device time) over all ranks."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def local_shard(row_ptr, col_idx, vals, world: int, rank: int, *, balance: str = "nnz", n: int = 0):
    """(plan, (row_ptr, col_idx, vals) of this rank's shard)."""
    rp_host = row_ptr.cpu().numpy() if isinstance(row_ptr, torch.Tensor) else row_ptr
    plan = plan_shards(rp_host, world, balance=balance, n=n)
    return plan, shard_csr(row_ptr, col_idx, vals, plan, rank)
