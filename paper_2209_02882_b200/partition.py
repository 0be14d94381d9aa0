"""nnz-balanced row shards for 1/2/4/8 GPUs.

A is cut into contiguous row blocks, B is replicated, C is row-disjoint, so a
sharded SpMM needs no collective; an optional gather of C lives in
``parallel.py``.  The cut points reuse the reference's partition primitive
``compute_block_starts`` (lowering.py:119-128) with chunk = ceil(nnz / k),
plus two fix-ups: ``starts[0] := 0`` (leading empty rows belong to shard 0)
and ``starts[k] := M`` (trailing empty rows belong to the last shard).  The
result is bit-exact integer output, pinned in tests/test_partition.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lowering import compute_block_starts

__all__ = ["ShardPlan", "shard_starts", "shard_starts_device", "bytes_balanced_starts",
           "plan_shards", "shard_csr"]


def shard_starts(row_ptr, k: int) -> np.ndarray:
    """int64[k+1] row cut points balancing nnz across k shards."""
    if k < 1:
        raise ValueError("shard count must be positive")
    rp = np.asarray(row_ptr, dtype=np.int64)
    m = rp.shape[0] - 1
    nnz = int(rp[-1])
    if nnz == 0:  # nothing to balance: split rows evenly
        return (np.arange(k + 1, dtype=np.int64) * m) // k
    chunk = -(-nnz // k)
    starts = compute_block_starts(rp, chunk, k)
    starts[0] = 0
    starts[k] = m
    return starts


def shard_starts_device(row_ptr, k: int):
    """``shard_starts`` on the device: the same cut points from the device
    block-start kernel (sgap_block_starts, lowering.compute_block_starts) and
    the two fix-ups; ``row_ptr`` is an int32 CUDA tensor, the result an int32
    CUDA tensor [k+1] (bit-identical to the host version, tests/test_gpu_parity)."""
    import torch

    from . import _native

    if k < 1:
        raise ValueError("shard count must be positive")
    m = int(row_ptr.numel()) - 1
    nnz = int(row_ptr[-1].item())
    if nnz == 0:
        return ((torch.arange(k + 1, dtype=torch.int64, device=row_ptr.device) * m) // k).to(torch.int32)
    out = torch.empty(k + 1, dtype=torch.int32, device=row_ptr.device)
    st = torch.cuda.current_stream(row_ptr.device).cuda_stream
    _native.check(_native.lib().sgap_block_starts(row_ptr.data_ptr(), m, -(-nnz // k), k,
                                                   out.data_ptr(), st), "sgap_block_starts")
    out[0] = 0
    out[k] = m
    return out


def bytes_balanced_starts(row_ptr, k: int, n: int) -> np.ndarray:
    """Cut points balancing 8*nnz + 4*n*rows (A stream + C write) instead of
    nnz alone -- for matrices whose nnz-balanced shards have very unequal row
    counts (unpermuted R-MAT)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    m = rp.shape[0] - 1
    weight = 8 * rp + 4 * n * np.arange(m + 1, dtype=np.int64)  # prefix weight up to row r
    total = int(weight[-1])
    targets = (np.arange(k + 1, dtype=np.int64) * total) // k
    starts = np.searchsorted(weight, targets, side="left").astype(np.int64)
    starts[0], starts[k] = 0, m
    return np.maximum.accumulate(np.minimum(starts, m))


def cost_balanced_starts(row_ptr, k: int, slice_starts, slice_costs) -> np.ndarray:
    """Cut points balancing a MEASURED cost: ``slice_starts`` (int[S+1] row
    cuts of S calibration slices, e.g. shard_starts(row_ptr, 64)) and
    ``slice_costs`` (S device times of each slice's SpMM on its own); cuts
    fall on slice boundaries where the cumulative cost crosses c*total/k.
    For matrices whose per-nonzero cost is far from uniform -- the
    unpermuted R-MAT, where low-id rows gather the L2-resident hot columns
    and high-id rows the cold ones, so nnz- and bytes-balanced shards differ
    2.6x in time (profiles/r02_scaling_projection_unpermuted_*.json)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    m = rp.shape[0] - 1
    ss = np.asarray(slice_starts, dtype=np.int64)
    cost = np.asarray(slice_costs, dtype=np.float64)
    if ss.shape[0] != cost.shape[0] + 1 or k < 1:
        raise ValueError("slice_starts must have one more entry than slice_costs")
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    out = np.empty(k + 1, dtype=np.int64)
    out[0], out[k] = 0, m
    for c in range(1, k):
        j = int(np.argmin(np.abs(cum - cum[-1] * c / k)))
        out[c] = ss[j]
    return np.maximum.accumulate(np.minimum(out, m))


@dataclass(frozen=True)
class ShardPlan:
    starts: np.ndarray          # int64[k+1] row cut points
    nnz_begin: np.ndarray       # int64[k] first position of each shard
    nnz_end: np.ndarray         # int64[k]

    @property
    def k(self) -> int:
        return int(self.starts.shape[0] - 1)

    def rows(self, g: int) -> tuple[int, int]:
        return int(self.starts[g]), int(self.starts[g + 1])

    def nnz(self, g: int) -> int:
        return int(self.nnz_end[g] - self.nnz_begin[g])


def plan_shards(row_ptr, k: int, *, balance: str = "nnz", n: int = 0,
                calibration=None) -> ShardPlan:
    """``balance``: "nnz" (the reference's compute_block_starts cuts),
    "bytes" (A stream + C write), or "cost" with ``calibration`` =
    (slice_starts, slice_costs) measured on the device."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    if balance == "nnz":
        s = shard_starts(rp, k)
    elif balance == "bytes":
        s = bytes_balanced_starts(rp, k, n)
    elif balance == "cost":
        if calibration is None:
            raise ValueError("balance='cost' needs calibration=(slice_starts, slice_costs)")
        s = cost_balanced_starts(rp, k, *calibration)
    else:
        raise ValueError(f"unknown balance {balance!r}")
    return ShardPlan(s, rp[s[:-1]], rp[s[1:]])


def shard_csr(row_ptr, col_idx, vals, plan: ShardPlan, g: int):
    """(row_ptr rebased to 0, col_idx slice, vals slice) of shard g; works on
    numpy arrays and torch tensors alike."""
    lo, hi = plan.rows(g)
    b, e = int(plan.nnz_begin[g]), int(plan.nnz_end[g])
    rp = row_ptr[lo:hi + 1] - b
    return rp, col_idx[b:e], vals[b:e]
