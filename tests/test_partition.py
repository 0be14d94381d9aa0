"""Multi-GPU host logic on CPU: nnz-balanced row shards (bit-exact against the
reference's partition primitive plus the documented fix-ups) and
the gloo world_size-2 plumbing (B broadcast, C gather of unequal slabs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2209_02882_b200 import generators as G
from paper_2209_02882_b200.matrices import random_csr
from paper_2209_02882_b200.parallel import broadcast_dense, gather_rows, max_over_ranks
from paper_2209_02882_b200.partition import (bytes_balanced_starts, plan_shards, shard_csr,
                                             shard_starts)


def _reference_cuts(row_ptr, k):
    rp = np.asarray(row_ptr, np.int64)
    nnz = int(rp[-1])
    s = oracle.block_starts(rp, -(-nnz // k), k)
    s[0], s[k] = 0, rp.shape[0] - 1
    return s


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_shard_cuts_bit_exact(k):
    for mat in (random_csr(300, 200, 0.05, 3), random_csr(64, 64, 0.5, 1)):
        assert shard_starts(mat.row_ptr, k).tolist() == _reference_cuts(mat.row_ptr, k).tolist()
    g = G.rmat(12, 16, seed=2, permute=False)
    rp = g.row_ptr.numpy()
    cuts = shard_starts(rp, k)
    assert cuts.tolist() == _reference_cuts(rp, k).tolist()
    plan = plan_shards(rp, k)
    assert int(plan.nnz_begin[0]) == 0 and int(plan.nnz_end[-1]) == g.nnz
    assert np.all(plan.nnz_end[:-1] == plan.nnz_begin[1:])
    # balance: no shard exceeds its ceil(nnz/k) share by more than one row
    lens = np.diff(rp)
    for gi in range(k):
        lo, hi = plan.rows(gi)
        slack = lens[hi] if hi < len(lens) else 0
        assert plan.nnz(gi) <= -(-g.nnz // k) + lens[lo:hi].max(initial=0) + slack


def test_leading_and_trailing_empty_rows_covered():
    rp = np.array([0, 0, 0, 3, 3, 7, 7, 7])
    for k in (1, 2, 3, 4):
        s = shard_starts(rp, k)
        assert s[0] == 0 and s[-1] == 7 and np.all(np.diff(s) >= 0)


def test_empty_matrix_splits_rows_evenly():
    s = shard_starts(np.zeros(11, np.int64), 4)
    assert s.tolist() == [0, 2, 5, 7, 10]


def test_bytes_balanced_cuts_are_monotone_and_cover():
    g = G.rmat(12, 16, seed=5, permute=False)
    rp = g.row_ptr.numpy()
    for k in (2, 4, 8):
        s = bytes_balanced_starts(rp, k, 128)
        assert s[0] == 0 and s[-1] == g.num_rows and np.all(np.diff(s) >= 0)


def test_sharded_product_equals_full_product():
    """Row shards with rebased row_ptr reproduce the full oracle product
    bitwise (rows are independent)."""
    a = random_csr(200, 150, 0.08, 9)
    b = np.random.default_rng(3).uniform(-1, 1, (150, 8))
    full = oracle.spmm_f64(a.row_ptr, a.col_idx, a.vals, b, 8)
    plan = plan_shards(a.row_ptr, 4)
    parts = []
    for gi in range(4):
        rp, ci, v = shard_csr(a.row_ptr, a.col_idx, a.vals, plan, gi)
        assert rp[0] == 0
        parts.append(oracle.spmm_f64(rp, ci, v, b, 8))
    assert np.array_equal(np.concatenate(parts), full)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = random_csr(120, 90, 0.1, 21)
        b = torch.zeros(90, 4, dtype=torch.float64)
        if rank == 0:
            b.copy_(torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, (90, 4))))
        broadcast_dense(b, src=0)
        plan = plan_shards(a.row_ptr, world)
        rp, ci, v = shard_csr(a.row_ptr, a.col_idx, a.vals, plan, rank)
        local = torch.from_numpy(oracle.spmm_f64(rp, ci, v, b.numpy(), 4))
        full = gather_rows(local, plan, root=0)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            want = oracle.spmm_f64(a.row_ptr, a.col_idx, a.vals, b.numpy(), 4)
            q.put((bool(np.array_equal(full.numpy(), want)), t))
        else:
            q.put((full is None, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_broadcast_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for ok, _ in results)
    assert all(t == 2.0 for _, t in results)


def test_cost_balanced_cuts_follow_measured_time():
    from paper_2209_02882_b200.partition import cost_balanced_starts, plan_shards
    rp = np.arange(0, 1001, dtype=np.int64) * 10      # 1000 rows, 10 nnz each
    slices = np.arange(0, 1001, 100, dtype=np.int64)  # 10 calibration slices
    costs = np.array([8, 1, 1, 1, 1, 1, 1, 1, 1, 4], dtype=np.float64)  # total 20
    s = cost_balanced_starts(rp, 2, slices, costs)
    assert list(s) == [0, 300, 1000]   # 8 + 1 + 1 = 10 of 20: the cut after the third slice
    s4 = cost_balanced_starts(rp, 4, slices, costs)
    assert s4[0] == 0 and s4[-1] == 1000 and np.all(np.diff(s4) >= 0)
    plan = plan_shards(rp, 2, balance="cost", calibration=(slices, costs))
    assert plan.rows(0) == (0, 300) and plan.nnz(0) == 3000
    with pytest.raises(ValueError):
        plan_shards(rp, 2, balance="cost")
