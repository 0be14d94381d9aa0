"""Small-matrix cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every family and every hardware walk of libsgap.so, the planner
and validation kernels, and the group primitives, each once on a matrix that
exercises hub rows (the float64 table, the error-free pass), empty rows and
ragged tails.  Checks results against the oracle so a sanitizer run is also
a parity run.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm, validate_csr  # noqa: E402
from paper_2209_02882_b200.lowering import KernelConfig, lower  # noqa: E402
from paper_2209_02882_b200.sim import exec_atomic_add_group, exec_seg_reduce_group  # noqa: E402
from paper_2209_02882_b200.space import parse_point  # noqa: E402
from paper_2209_02882_b200.templates import algorithm_template  # noqa: E402


class _Rp:
    def __init__(self, m, k, rp):
        self.num_rows, self.num_cols, self.row_ptr = m, k, rp


def matrix(seed=3):
    rng = np.random.default_rng(seed)
    m, k = 300, 6000
    lens = rng.integers(0, 40, m)
    lens[::11] = 0
    lens[7] = 5000   # > kExactRow: the error-free pass / float64 products
    lens[40] = 900   # long row: the float64 table
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(k, int(L), replace=False)) for L in lens if L])
    vals = rng.uniform(-1, 1, rp[-1])
    return m, k, rp, cols, vals


def main():
    dev = torch.device("cuda", 0)
    m, k, rp, cols, vals = matrix()
    a = DeviceCsr(m, k, torch.from_numpy(rp.astype(np.int32)).to(dev),
                  torch.from_numpy(cols.astype(np.int32)).to(dev),
                  torch.from_numpy(vals.astype(np.float32)).to(dev))
    assert validate_csr(a) is None
    cases = [
        ("nnz:64,col:4,r:1", 256, 1), ("nnz:64,col:4,r:1", 256, 5), ("nnz:64,col:4,r:1", 256, 9),
        ("nnz:1,col:4,r:8", 1024, 1), ("nnz:1,col:4,r:1", 256, 1),
        ("row:4,col:4,r:1", 256, 6), ("row:4,col:4,r:1", 256, 7),
        ("nnz:64,col:4,r:1", 256, 2), ("nnz:256,col:4,r:1", 1024, 3),
        ("nnz:256,col:4,r:1", 1024, 4), ("nnz:6,col:1,r:1", 256, 1), ("nnz:512,col:4,r:1", 256, 1),
        ("nnz:1,col:4,r:8", 1024, 0), ("nnz:1,col:4,r:1", 256, 0), ("nnz:1,col:1,r:32", 1024, 0),
        ("row:1,col:4,r:1", 256, 0), ("row:4,col:4,r:1", 256, 2), ("row:4,col:4,r:1", 256, 3),
        ("row:4,col:4,r:1", 256, 4), ("row:1/8,col:4,r:8", 256, 0), ("row:1/32,col:1,r:32", 256, 0),
        ("row:4,col:4,r:1", 256, 8),
    ]
    for n in (128, 64, 40):
        b = torch.rand((k, n), device=dev) * 2 - 1
        for prec in (torch.float32, torch.float64):
            aa = DeviceCsr(m, k, a.row_ptr, a.col_idx, a.vals.to(prec))
            bb = b.to(prec)
            want = oracle.spmm_f64(rp.astype(np.int32), cols.astype(np.int32),
                                   aa.vals.cpu().numpy(), bb.cpu().numpy(), n)
            c = torch.empty((m, n), dtype=prec, device=dev)
            for text, p, variant in cases:
                tpl = algorithm_template(parse_point(text), KernelConfig(n=n, p=p))
                if tpl is None:
                    continue
                if variant in (3, 4) and text.startswith("row") and not (
                        (n // tpl.c) % 32 == 0 or (n // tpl.c) in (2, 4, 8, 16)):
                    continue
                if variant in (3, 4) and text.startswith("nnz") and (n // tpl.c) < 32:
                    continue
                if variant == 8 and not ((n // tpl.c) % 32 == 0 or n // tpl.c == 16):
                    continue
                kk = lower(tpl, _Rp(m, k, rp), compute_starts=False)
                aux = prepare_aux(kk, aa, validate=True, l2_hints=True)
                if variant in (6, 7) and not aux.plan.aux.d_union_off4:
                    continue  # rows > 64: no union plan (the hub rows of this matrix)
                for acc in (False, True):
                    c.zero_() if acc else c.fill_(float("nan"))
                    spmm(kk, aa, bb, c, aux=aux, accumulate=acc, hw_variant=variant)
                    err = oracle.max_rel_error(c.cpu().numpy(), want)
                    tol = 1e-5 if prec == torch.float32 else 1e-12
                    assert err <= tol, (text, variant, n, prec, acc, err)
            print("n", n, "ok")
    # the row-blocked union walk (row-multiple variants 6/7) needs rows <= 64:
    # a banded matrix with empty rows and M not a multiple of 8
    rng = np.random.default_rng(5)
    m2, k2 = 203, 480  # columns up to 2*202 - 40 + 79 = 443
    lens2 = rng.integers(0, 30, m2)
    lens2[::13] = 0
    rp2 = np.concatenate([[0], np.cumsum(lens2)]).astype(np.int64)
    cols2 = np.concatenate([np.sort(rng.choice(np.arange(max(0, i * 2 - 40), max(0, i * 2 - 40) + 80),
                                               int(L), replace=False)) for i, L in enumerate(lens2) if L])
    a2 = DeviceCsr(m2, k2, torch.from_numpy(rp2.astype(np.int32)).to(dev),
                   torch.from_numpy(cols2.astype(np.int32)).to(dev),
                   torch.from_numpy(rng.uniform(-1, 1, rp2[-1]).astype(np.float32)).to(dev))
    b2 = torch.rand((k2, 128), device=dev) * 2 - 1
    want2 = oracle.spmm_f64(rp2.astype(np.int32), cols2.astype(np.int32), a2.vals.cpu().numpy(),
                            b2.cpu().numpy(), 128)
    c2 = torch.empty((m2, 128), device=dev)
    for variant in (6, 7):
        kk = lower(algorithm_template(parse_point("row:4,col:4,r:1"), KernelConfig(n=128, p=256)),
                   _Rp(m2, k2, rp2), compute_starts=False)
        aux = prepare_aux(kk, a2, validate=True)
        c2.fill_(float("nan"))
        spmm(kk, a2, b2, c2, aux=aux, hw_variant=variant)
        assert oracle.max_rel_error(c2.cpu().numpy(), want2) <= 1e-5, variant
    print("union walk ok")
    # column-panel walk (nnz-multiple variant 10): B must exceed the L2 for
    # the planner to cut panels -- 140,000 x 256 float32 (143 MB) gives
    # 64-column panels (4 passes); hub row, float64 table and empty rows kept
    m3, k3, n3 = 300, 140_000, 256
    rng = np.random.default_rng(9)
    lens3 = rng.integers(0, 40, m3)
    lens3[::11] = 0
    lens3[7], lens3[40] = 5000, 900
    rp3 = np.concatenate([[0], np.cumsum(lens3)]).astype(np.int64)
    cols3 = np.concatenate([np.sort(rng.choice(k3, int(L), replace=False)) for L in lens3 if L])
    a3 = DeviceCsr(m3, k3, torch.from_numpy(rp3.astype(np.int32)).to(dev),
                   torch.from_numpy(cols3.astype(np.int32)).to(dev),
                   torch.from_numpy(rng.uniform(-1, 1, rp3[-1]).astype(np.float32)).to(dev))
    b3 = torch.rand((k3, n3), device=dev) * 2 - 1
    want3 = oracle.spmm_f64(rp3.astype(np.int32), cols3.astype(np.int32), a3.vals.cpu().numpy(),
                            b3.cpu().numpy(), n3)
    c3 = torch.empty((m3, n3), device=dev)
    for text in ("nnz:64,col:4,r:1", "nnz:512,col:4,r:1"):
        kk = lower(algorithm_template(parse_point(text), KernelConfig(n=n3, p=1024)),
                   _Rp(m3, k3, rp3), compute_starts=False)
        aux = prepare_aux(kk, a3, validate=True)
        assert aux.plan.aux.panel_lanes == 16, aux.plan.aux.panel_lanes
        for acc in (False, True):
            c3.zero_() if acc else c3.fill_(float("nan"))
            spmm(kk, a3, b3, c3, aux=aux, accumulate=acc, hw_variant=10)
            assert oracle.max_rel_error(c3.cpu().numpy(), want3) <= 1e-5, (text, acc)
    del b3
    print("column-panel walk ok")
    # shifted-block walk (row-multiple variant 8) on a stencil: shifted blocks,
    # grid-edge fallback blocks, N/c = 32, 64 (two panels) and 16 (lane groups)
    from paper_2209_02882_b200 import generators as G
    st = G.stencil27(12, device=dev)
    a4 = DeviceCsr(st.num_rows, st.num_cols, st.row_ptr.to(torch.int32), st.col_idx.to(torch.int32),
                   st.vals.to(torch.float32))
    rp4 = a4.row_ptr.cpu().numpy().astype(np.int64)
    for n in (128, 256, 64):
        b4 = torch.rand((st.num_cols, n), device=dev) * 2 - 1
        want4 = oracle.spmm_f64(rp4.astype(np.int32), a4.col_idx.cpu().numpy(), a4.vals.cpu().numpy(),
                                b4.cpu().numpy(), n)
        kk = lower(algorithm_template(parse_point("row:8,col:4,r:1"), KernelConfig(n=n, p=256)),
                   _Rp(st.num_rows, st.num_cols, rp4), compute_starts=False)
        aux = prepare_aux(kk, a4, validate=True)
        c4 = torch.full((st.num_rows, n), float("nan"), device=dev)
        spmm(kk, a4, b4, c4, aux=aux, hw_variant=8)
        assert oracle.max_rel_error(c4.cpu().numpy(), want4) <= 1e-5, n
    print("shifted-block walk ok")
    # group primitives
    out = np.zeros(16)
    assert exec_seg_reduce_group(np.array([5, 5, 7, 7]), np.array([1.0, 2, 3, 4]), out, group_size=4) == 2
    out = np.zeros(8)
    assert exec_atomic_add_group(np.array([3, 3, 3, 3]), np.ones(4), out, group_size=4) == 1
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
