"""The reference compiler's emitted kernels (baseline/refgen): the frozen
manifest agrees with this package's planner, the launch library loads and
holds every text at float32 and float64; on the GPU each kernel matches the
CPU oracle (which also checks the group-macro bodies written for them)."""

import json

import numpy as np
import pytest
import torch

import oracle
from baseline import refgen
from paper_2209_02882_b200.device import DeviceCsr, device_block_starts
from paper_2209_02882_b200.lowering import KernelConfig
from paper_2209_02882_b200.matrices import random_csr, random_dense
from paper_2209_02882_b200.runner import build_kernel
from paper_2209_02882_b200.space import parse_point

from conftest import GOLDEN


def test_manifest_matches_planner():
    ks = refgen.kernels()
    assert len(ks) == 171
    m = random_csr(64, 64, 0.0625, seed=1)
    for rk in ks:
        k = build_kernel(parse_point(rk.point), KernelConfig(n=rk.n, p=rk.p), m)
        assert k is not None, rk.point
        assert (k.family, k.block_size) == (rk.family, rk.block_size), rk.point
        assert (GOLDEN / "refgen" / f"{rk.id}.cu").exists()
    corners = {rk.point for rk in ks if rk.da_spmm_corner}
    assert corners == {"nnz:32,col:1,r:1", "row:1,col:1,r:1", "row:1/32,col:1,r:32",
                       "nnz:1,col:1,r:32"}
    ids = {rk.id for rk in ks}
    assert refgen.lib().refgen_count() == 2 * len(ids)
    assert refgen.lib().refgen_launch(b"nope", 0, 1, 32, None, None, None, None, None, None,
                                      1, 1, None) == -1


def _device(mat, dtype, dev):
    return DeviceCsr(mat.num_rows, mat.num_cols,
                     torch.as_tensor(np.asarray(mat.row_ptr, np.int32), device=dev),
                     torch.as_tensor(np.asarray(mat.col_idx, np.int32), device=dev),
                     torch.as_tensor(np.asarray(mat.vals), dtype=dtype, device=dev))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [4, 32, 128])
def test_reference_kernels_match_oracle(n):
    """Every frozen kernel at this n on a 1%-like random matrix, float64
    (<= 1e-12) and float32 (<= 1e-4, the reference's default tolerance,
    runner.py:165-206: its kernels sum in the value type)."""
    dev = torch.device("cuda", 0)
    mat = random_csr(700, 500, 0.02, seed=5)
    b = random_dense(500, n, seed=6)
    want = oracle.spmm_f64(np.asarray(mat.row_ptr, np.int32), np.asarray(mat.col_idx, np.int32),
                           np.asarray(mat.vals, np.float64),
                           np.asarray(b.vals, np.float64).reshape(500, n), n)
    want32 = oracle.spmm_f64(np.asarray(mat.row_ptr, np.int32), np.asarray(mat.col_idx, np.int32),
                             np.asarray(mat.vals, np.float32),
                             np.asarray(b.vals, np.float32).reshape(500, n), n)
    count = 0
    for rk in refgen.kernels():
        if rk.n != n:
            continue
        k = build_kernel(parse_point(rk.point), KernelConfig(n=n, p=rk.p), mat)
        for dtype, tol, ref in ((torch.float64, 1e-12, want), (torch.float32, 1e-4, want32)):
            a = _device(mat, dtype, dev)
            bt = torch.as_tensor(np.asarray(b.vals).reshape(500, n), dtype=dtype, device=dev)
            c = torch.empty((mat.num_rows, n), dtype=dtype, device=dev)
            starts = device_block_starts(a, k.chunk, k.grid_size) if rk.has_block_starts else None
            refgen.run(rk, k.grid_size, a, bt, c, starts)
            err = oracle.max_rel_error(c.cpu().numpy(), ref)
            assert err <= tol, (rk.point, n, str(dtype), err)
        count += 1
    assert count > 0
