"""Parity at BASELINE sizes: config 2 (R-MAT scale 20, 16.09M nnz, N=128)
and a 27-point stencil, every family, against the CPU oracle.

Power-law hub rows (up to ~40k nonzeros) are where float32 accumulation
breaks the 1e-5 bound unless long sums are carried in float64 -- this is the
test that pins the engine's numerics policy."""

import numpy as np
import pytest
import torch

import oracle
from paper_2209_02882_b200 import generators as G
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm
from paper_2209_02882_b200.lowering import KernelConfig, lower
from paper_2209_02882_b200.space import parse_point
from paper_2209_02882_b200.templates import algorithm_template

pytestmark = pytest.mark.gpu

TOL = 1e-5

POINTS_N128 = [
    ("nnz:32,col:4,r:1", 256), ("nnz:8,col:2,r:1", 1024), ("nnz:32,col:1,r:1", 4096),
    ("nnz:1,col:4,r:8", 1024), ("nnz:1,col:4,r:32", 1024), ("nnz:1,col:4,r:1", 256),
    ("row:1,col:4,r:1", 256), ("row:4,col:1,r:1", 256),
    ("row:1/4,col:4,r:4", 256), ("row:1/32,col:4,r:32", 256),
]


class _Rp:
    def __init__(self, m, k, rp):
        self.num_rows, self.num_cols, self.row_ptr = m, k, rp


def _device(g):
    return DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
                     g.vals.to(torch.float32))


def _check(g, n, points):
    dev = torch.device("cuda", 0)
    a = _device(g)
    gen = torch.Generator(device=dev)
    gen.manual_seed(2)
    b = torch.rand((g.num_cols, n), generator=gen, device=dev) * 2 - 1
    rp = a.row_ptr.cpu().numpy()
    want = oracle.spmm_f64(rp, a.col_idx.cpu().numpy(), a.vals.cpu().numpy(), b.cpu().numpy(), n)
    c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
    worst = {}
    for item in points:
        text, p = item[:2]
        hw_variant = item[2] if len(item) > 2 else 0
        split_rows = item[3] if len(item) > 3 else False
        tpl = algorithm_template(parse_point(text), KernelConfig(n=n, p=p))
        assert tpl is not None, text
        k = lower(tpl, _Rp(a.num_rows, a.num_cols, rp.astype(np.int64)), compute_starts=False)
        c.fill_(float("nan"))
        spmm(k, a, b, c, aux=prepare_aux(k, a, split_rows=split_rows), hw_variant=hw_variant)
        err = oracle.max_rel_error(c.cpu().numpy(), want)
        worst[item] = err
        assert err <= TOL, (item, err)
    return worst


def test_config2_rmat_every_family():
    g = G.rmat(20, 16, seed=1, device="cuda")
    assert g.nnz > 16_000_000
    print(_check(g, 128, POINTS_N128))


def test_config2_long_chunk_walks():
    """The bench's schedules (long chunks, g up to 2048) on every walk
    variant, with and without split-row routing to the float64 table."""
    g = G.rmat(20, 16, seed=1, device="cuda")
    pts = [(t, 256, v, split) for t in ("nnz:512,col:4,r:1", "nnz:2048,col:4,r:1", "nnz:128,col:4,r:1")
           for v in (1, 3, 4, 5) for split in (False, True)]
    # nnz-one's segment groups as a serial walk (variant 1), hub rows in the table
    pts += [("nnz:1,col:4,r:8", 1024, 1, False), ("nnz:1,col:4,r:32", 1024, 1, False),
            ("nnz:1,col:4,r:1", 256, 1, False)]
    pts += [("nnz:128,col:4,r:1", 256, 2, False), ("nnz:64,col:2,r:1", 1024, 3, True)]
    print(_check(g, 128, pts))


def test_config3_reddit_shaped():
    """BASELINE config 3 (Chung-Lu, 233k rows, 114.5M nnz, hub rows of tens
    of thousands of nonzeros) at N=64: the rows where float32 product
    rounding alone exceeds 1e-5 without the error-free accumulate."""
    g = G.config_matrix(3, device="cuda")
    print(_check(g, 64, [("nnz:512,col:4,r:1", 256, 1), ("nnz:128,col:2,r:1", 1024, 3),
                         ("nnz:32,col:4,r:1", 256, 2), ("row:4,col:2,r:1", 256, 4),
                         ("row:1,col:4,r:1", 256, 2), ("row:1/4,col:4,r:4", 256),
                         ("nnz:1,col:4,r:1", 256), ("nnz:1,col:2,r:8", 256)]))


def test_row_staged_variants():
    """Row-multiple with a warp per row (hw variants 3/4, N/c == 32): stencil
    rows (<= 27, the float32 path) and R-MAT hub rows (> 64, the float64
    path) at N = 128 / 64 / 32; at N/c = 64 / 128 (N = 256, 512), one pass
    per 32c-column panel of B and C in place; at N/c = 16 / 8 / 4 / 2, 2 / 4 / 8 / 16
    rows per warp."""
    st = G.stencil27(64, device="cuda")
    rm = G.rmat(16, 16, seed=5, device="cuda")
    for g in (st, rm):
        print(_check(g, 128, [("row:4,col:4,r:1", 256, 3), ("row:4,col:4,r:1", 256, 4),
                              ("row:1,col:4,r:1", 256, 4), ("row:16,col:4,r:1", 256, 4)]))
        print(_check(g, 64, [("row:4,col:2,r:1", 256, 4), ("row:2,col:2,r:1", 256, 3)]))
        print(_check(g, 32, [("row:4,col:1,r:1", 256, 4)]))
        print(_check(g, 256, [("row:8,col:4,r:1", 256, 4), ("row:4,col:2,r:1", 256, 3),
                              ("row:2,col:4,r:1", 1024, 3)]))
        print(_check(g, 512, [("row:8,col:4,r:1", 256, 4)]))
        # N/c = 16 / 8: 2 / 4 rows per warp (R-MAT hub rows take the per-lane walk)
        print(_check(g, 64, [("row:8,col:4,r:1", 1024, 4), ("row:4,col:4,r:1", 256, 3)]))
        print(_check(g, 32, [("row:8,col:4,r:1", 256, 4), ("row:4,col:2,r:1", 256, 3)]))
        print(_check(g, 16, [("row:4,col:2,r:1", 256, 4), ("row:8,col:4,r:1", 256, 4)]))
        print(_check(g, 8, [("row:4,col:4,r:1", 256, 4)]))  # 2 lanes per row
    # N/c not a multiple of 32 (N = 192: 48 lanes): refused
    k = lower(algorithm_template(parse_point("row:4,col:4,r:1"), KernelConfig(n=192, p=192)),
              _Rp(st.num_rows, st.num_cols, st.row_ptr.cpu().numpy().astype(np.int64)),
              compute_starts=False)
    a = _device(st)
    from paper_2209_02882_b200 import _native
    with pytest.raises(_native.SgapError):
        spmm(k, a, torch.zeros((a.num_cols, 192), device="cuda"),
             torch.empty((a.num_rows, 192), device="cuda"), aux=prepare_aux(k, a), hw_variant=4)


def test_stencil_small_n():
    g = G.stencil27(48, device="cuda")
    assert g.nnz == (3 * 48 - 2) ** 3
    pts = [("nnz:1,col:1,r:8", 256), ("nnz:1,col:4,r:4", 256), ("nnz:32,col:4,r:1", 256),
           ("row:1,col:4,r:1", 256), ("row:1/8,col:1,r:8", 256), ("row:1/4,col:4,r:4", 256)]
    print(_check(g, 4, pts))


def test_unpermuted_rmat_small_n():
    g = G.rmat(16, 16, seed=3, permute=False, device="cuda")
    pts = [("nnz:1,col:4,r:32", 1024), ("nnz:1,col:1,r:1", 256), ("nnz:16,col:4,r:1", 256),
           ("row:1,col:4,r:1", 256), ("row:1/32,col:1,r:32", 256)]
    print(_check(g, 8, pts))


def test_pipelined_host_spmm_matches_single_call():
    from paper_2209_02882_b200.pipeline import HostSpmm
    from paper_2209_02882_b200.selector import Candidate, plan_for

    g = G.rmat(16, 16, seed=4, device="cuda")
    a = _device(g)
    n = 64
    b = (torch.rand((a.num_cols, n), device="cuda") * 2 - 1)
    h_rp, h_ci, h_v = (x.cpu().pin_memory() for x in (a.row_ptr, a.col_idx, a.vals))
    h_b = b.cpu().pin_memory()
    want = oracle.spmm_f64(h_rp.numpy(), h_ci.numpy(), h_v.numpy(), h_b.numpy(), n)
    for point, p, blocks in (("nnz:128,col:4,r:1", 256, 5), ("row:1,col:4,r:1", 256, 3),
                             ("nnz:1,col:4,r:8", 1024, 4)):
        cand = Candidate(point, p)
        pipe = HostSpmm(a.num_rows, a.num_cols, n, h_rp, h_ci,
                        lambda rows, rp: plan_for(cand, n, rows, a.num_cols, rp), blocks=blocks)
        for _ in range(3):  # back-to-back calls exercise both buffer sets
            h_c = torch.full((a.num_rows, n), float("nan")).pin_memory()
            pipe(h_v, h_b, h_c)
            pipe.wait()
            torch.cuda.synchronize()
            assert oracle.max_rel_error(h_c.numpy(), want) <= TOL, point


def test_config5_rmat_scale24_sampled_rows():
    """BASELINE config 5 (R-MAT scale 24, ~257M nnz, N=128) at full size on one
    GPU: the best EB schedule against the oracle on a sample of rows
    (including the heaviest ones) -- a full CPU oracle pass would need ~35 GB
    of host memory."""
    g = G.rmat(24, 16, seed=1, device="cuda")
    assert g.nnz > 250_000_000
    a = _device(g)
    del g
    torch.cuda.empty_cache()
    n = 128
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2)
    b = torch.rand((a.num_cols, n), generator=gen, device="cuda") * 2 - 1
    c = torch.empty((a.num_rows, n), dtype=torch.float32, device="cuda")
    rp = a.row_ptr.cpu().numpy()
    tpl = algorithm_template(parse_point("nnz:512,col:4,r:1"), KernelConfig(n=n, p=256))
    k = lower(tpl, _Rp(a.num_rows, a.num_cols, rp.astype(np.int64)), compute_starts=False)
    spmm(k, a, b, c, aux=prepare_aux(k, a))
    lens = np.diff(rp)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([np.argsort(-lens)[:64], rng.integers(0, a.num_rows, 4000)]))
    sub_rp = np.concatenate([[0], np.cumsum(lens[rows])]).astype(np.int32)
    sel = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    ci = a.col_idx.cpu().numpy()[sel]
    vals = a.vals.cpu().numpy()[sel]
    want = oracle.spmm_f64(sub_rp, ci, vals, b.cpu().numpy(), n)
    got = c[torch.from_numpy(rows).cuda()].cpu().numpy()
    err = oracle.max_rel_error(got, want)
    assert err <= TOL, err
    print("config5 sampled rows", rows.size, "max_rel_error", err)


def test_exact_rows_and_empty_row_gaps():
    """Rows beyond the error-free threshold (here > 65,536 nonzeros) next to
    empty rows at the start, middle and end of the matrix: the owner-mode walk
    zero-fills every empty row itself, including around chunks that the
    exact-row path takes over."""
    rng = np.random.default_rng(11)
    m, k, n = 64, 100_000, 128
    lens = np.zeros(m, dtype=np.int64)
    lens[5] = 70_001      # exact row after 5 leading empty rows
    lens[9:20] = rng.integers(1, 40, 11)
    lens[30] = 66_000     # exact row followed by empty rows to the end
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(k, size=L, replace=False)) for L in lens if L])
    vals = rng.uniform(-1, 1, rp[-1])
    import types
    g = types.SimpleNamespace(num_rows=m, num_cols=k, row_ptr=torch.from_numpy(rp).cuda(),
                              col_idx=torch.from_numpy(cols).cuda(),
                              vals=torch.from_numpy(vals).cuda())
    a = _device(g)
    b = torch.rand((k, n), device="cuda") * 2 - 1
    want = oracle.spmm_f64(a.row_ptr.cpu().numpy(), a.col_idx.cpu().numpy(), a.vals.cpu().numpy(),
                           b.cpu().numpy(), n)
    c = torch.empty((m, n), dtype=torch.float32, device="cuda")
    # every family and walk over the error-free rows: EB register walk
    # (inline float64 chunks), TMA and lane-staged walks (k_nnz_multiple_exact
    # overlapped by programmatic dependent launch), nnz-one (float64 table
    # sums), RB walks (float64 products per row), row-reciprocal groups
    for text, p, variant in (("nnz:512,col:4,r:1", 256, 1), ("nnz:512,col:4,r:1", 256, 5),
                             ("nnz:64,col:4,r:1", 1024, 2),
                             ("nnz:32,col:4,r:1", 256, 1), ("nnz:256,col:4,r:1", 256, 3),
                             ("nnz:1,col:4,r:8", 1024, 0), ("nnz:1,col:4,r:1", 256, 0),
                             ("row:1,col:4,r:1", 256, 0), ("row:4,col:4,r:1", 256, 2),
                             ("row:4,col:4,r:1", 256, 4), ("row:1/8,col:4,r:8", 256, 0),
                             ("row:1/32,col:1,r:32", 256, 0)):
        tpl = algorithm_template(parse_point(text), KernelConfig(n=n, p=p))
        kk = lower(tpl, _Rp(m, k, rp), compute_starts=False)
        aux = prepare_aux(kk, a)
        if kk.family == "nnz-multiple":
            assert aux.has_exact_rows == 1
        c.fill_(float("nan"))
        spmm(kk, a, b, c, aux=aux, hw_variant=variant)
        got = c.cpu().numpy()
        assert not np.isnan(got).any(), text
        assert oracle.max_rel_error(got, want) <= TOL, text


@pytest.mark.parametrize("variant", [6, 7])
def test_row_blocked_union_walk(variant):
    """Row-multiple hw variants 6/7: a warp per 4/8-row block walking the
    union of the block's columns (plan-time k_union_rows).  Stencils, a
    banded matrix with empty rows and M not a multiple of the block, both
    precisions, overwrite and accumulate; matrices with rows > 64 are
    rejected (SGAP_ERR_ARG) rather than run."""
    from paper_2209_02882_b200 import _native
    rng = np.random.default_rng(variant)
    m, k = 10_003, 9_000
    lens = rng.integers(0, 40, m)
    lens[::17] = 0
    rows, cols = [], []
    for i, L in enumerate(lens):
        lo = max(0, min(k - 80, i * k // m - 40))
        cs = np.sort(rng.choice(np.arange(lo, lo + 80), int(L), replace=False))
        rows.append(np.full(L, i))
        cols.append(cs)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    import types
    band = types.SimpleNamespace(num_rows=m, num_cols=k, row_ptr=torch.from_numpy(rp).cuda(),
                                 col_idx=torch.from_numpy(np.concatenate(cols)).cuda(),
                                 vals=torch.from_numpy(rng.uniform(-1, 1, rp[-1])).cuda())
    for g in (G.stencil27(40, device="cuda"), band):
        print(_check(g, 128, [("row:4,col:4,r:1", 256, variant), ("row:1,col:4,r:1", 256, variant)]))
        print(_check(g, 64, [("row:2,col:2,r:1", 256, variant)]))
        print(_check(g, 32, [("row:4,col:1,r:1", 256, variant)]))
    # float64 and accumulate mode
    a = _device(band)
    a64 = DeviceCsr(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, band.vals.to(torch.float64))
    b = torch.rand((k, 128), dtype=torch.float64, device="cuda") * 2 - 1
    c = torch.ones((m, 128), dtype=torch.float64, device="cuda")
    tpl = algorithm_template(parse_point("row:4,col:4,r:1"), KernelConfig(n=128, p=256))
    kk = lower(tpl, _Rp(m, k, rp), compute_starts=False)
    spmm(kk, a64, b, c, aux=prepare_aux(kk, a64), accumulate=True, hw_variant=variant)
    want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(), a64.vals.cpu().numpy(),
                           b.cpu().numpy(), 128) + 1.0
    assert oracle.max_rel_error(c.cpu().numpy(), want) <= 1e-12
    # rows longer than 64: no union plan, the variant refuses
    rm = G.rmat(14, 16, seed=2, device="cuda")
    ar = _device(rm)
    kr = lower(tpl, _Rp(ar.num_rows, ar.num_cols, ar.row_ptr.cpu().numpy().astype(np.int64)),
               compute_starts=False)
    cr = torch.empty((ar.num_rows, 128), device="cuda")
    br = torch.rand((ar.num_cols, 128), device="cuda")
    with pytest.raises(_native.SgapError):
        spmm(kr, ar, br, cr, aux=prepare_aux(kr, ar), hw_variant=variant)


def test_shifted_block_walk_bitwise():
    """Row-multiple hw variant 8 (shifted 4-row blocks, gathers shared
    across the block) give C bit-identical to the warp-per-row walk (variant
    4): each row is summed serially in CSR order either way, and blocks that
    are not shifted copies (grid edges, ragged or long rows, M not a multiple
    of the block) take that walk inline.  Stencil, a band with empty rows,
    a tridiagonal-plus-hub matrix, N/c = 32 and 64 (column panels), float32
    and float64, overwrite and accumulate; also against the oracle."""
    import types
    variant = 8
    rng = np.random.default_rng(variant)
    # band with ragged rows (few shifted blocks) and empty rows
    m, k = 10_003, 9_000
    lens = rng.integers(0, 40, m)
    lens[::17] = 0
    cols = []
    for i, L in enumerate(lens):
        lo = max(0, min(k - 80, i * k // m - 40))
        cols.append(np.sort(rng.choice(np.arange(lo, lo + 80), int(L), replace=False)))
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    band = types.SimpleNamespace(num_rows=m, num_cols=k, row_ptr=torch.from_numpy(rp).cuda(),
                                 col_idx=torch.from_numpy(np.concatenate(cols)).cuda(),
                                 vals=torch.from_numpy(rng.uniform(-1, 1, rp[-1])).cuda())
    # tridiagonal rows (shifted blocks) with runs of 1/2/4/5 and a few hub rows
    m2 = 5_001
    offs = np.array([-700, -3, -2, -1, 0, 1, 5, 6, 7, 8, 9, 300])
    rows2, cols2 = [], []
    for i in range(m2):
        cs = i + offs
        cs = cs[(cs >= 0) & (cs < m2)]
        if i % 1000 == 500:  # a hub row longer than 64 (float64 path inline)
            cs = np.unique(np.concatenate([cs, rng.choice(m2, 300, replace=False)]))
        rows2.append(np.full(cs.size, i))
        cols2.append(cs)
    lens2 = np.array([c.size for c in cols2])
    rp2 = np.concatenate([[0], np.cumsum(lens2)]).astype(np.int64)
    tri = types.SimpleNamespace(num_rows=m2, num_cols=m2, row_ptr=torch.from_numpy(rp2).cuda(),
                                col_idx=torch.from_numpy(np.concatenate(cols2)).cuda(),
                                vals=torch.from_numpy(rng.uniform(-1, 1, rp2[-1])).cuda())
    for g in (G.stencil27(40, device="cuda"), band, tri):
        for n, c in ((128, 4), (256, 4), (64, 2), (64, 4), (32, 4)):
            for dt, tol in ((torch.float32, TOL), (torch.float64, 1e-12)):
                a0 = _device(g)
                a = DeviceCsr(a0.num_rows, a0.num_cols, a0.row_ptr, a0.col_idx, g.vals.to(dt))
                rph = a.row_ptr.cpu().numpy().astype(np.int64)
                b = torch.rand((a.num_cols, n), dtype=dt, device="cuda") * 2 - 1
                tpl = algorithm_template(parse_point(f"row:8,col:{c},r:1"),
                                         KernelConfig(n=n, p=256))
                kk = lower(tpl, _Rp(a.num_rows, a.num_cols, rph), compute_starts=False)
                outs = []
                for v in (4, variant):
                    for acc in (False, True):
                        cc = torch.full((a.num_rows, n), 0.5, dtype=dt, device="cuda")
                        spmm(kk, a, b, cc, aux=prepare_aux(kk, a), accumulate=acc, hw_variant=v)
                        outs.append(cc)
                assert torch.equal(outs[0], outs[2]) and torch.equal(outs[1], outs[3]), (n, c, dt)
                want = oracle.spmm_f64(rph.astype(np.int32), a.col_idx.cpu().numpy(),
                                       a.vals.cpu().numpy(), b.cpu().numpy(), n)
                assert oracle.max_rel_error(outs[2].cpu().numpy(), want) <= tol
                assert oracle.max_rel_error(outs[3].cpu().numpy(), want + 0.5) <= tol
    # N/c not 8, 16 or a multiple of 32: refused (SGAP_ERR_ARG)
    from paper_2209_02882_b200 import _native
    a = _device(tri)
    tpl = algorithm_template(parse_point("row:8,col:4,r:1"), KernelConfig(n=16, p=256))
    kk = lower(tpl, _Rp(a.num_rows, a.num_cols, rp2), compute_starts=False)
    with pytest.raises(_native.SgapError):
        spmm(kk, a, torch.rand((m2, 16), device="cuda"), torch.empty((m2, 16), device="cuda"),
             aux=prepare_aux(kk, a), hw_variant=variant)


def test_cold_column_hint_walk():
    """hw variant 9: the row_ptr walk reading the plan's flagged col_idx copy
    (bit 31 = cold column, gathered with the streaming cache operator):
    same results as variant 1, the hints never leak into an index --
    including chunks inside error-free hub rows (the inline float64 path)."""
    g = G.rmat(17, 16, seed=6, device="cuda")
    a = _device(g)
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    n = 128
    b = torch.rand((a.num_cols, n), device="cuda") * 2 - 1
    want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(), a.vals.cpu().numpy(),
                           b.cpu().numpy(), n)
    c = torch.empty((a.num_rows, n), device="cuda")
    for text, p in (("nnz:512,col:4,r:1", 256), ("nnz:32,col:4,r:1", 256)):
        k = lower(algorithm_template(parse_point(text), KernelConfig(n=n, p=p)),
                  _Rp(a.num_rows, a.num_cols, rp), compute_starts=False)
        aux = prepare_aux(k, a, l2_hints=True)
        assert aux.plan.aux.d_col_hinted
        wb = {}
        for v in (1, 9):
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            c.fill_(float("nan"))
            spmm(k, a, b, c, aux=aux, hw_variant=v, writebacks=cnt)
            assert oracle.max_rel_error(c.cpu().numpy(), want) <= TOL, (text, v)
            wb[v] = int(cnt.item())
        assert wb[1] == wb[9]
        # without hints in the plan, variant 9 refuses
        from paper_2209_02882_b200 import _native
        with pytest.raises(_native.SgapError):
            spmm(k, a, b, c, aux=prepare_aux(k, a, l2_hints=False), hw_variant=9)


def test_column_panel_walk():
    """hw variant 10: the row_ptr walk in column-panel order (every chunk for
    one panel of B's columns, then the next panel) when B exceeds the L2 but a
    panel fits half of it.  Same results and writeback counts as variant 1
    on a Chung-Lu matrix with config 3's column count (64-column panels) and
    an R-MAT one at N = 512 (32-column panels, 16 passes), hub rows included;
    refused when all of B fits the L2."""
    from paper_2209_02882_b200 import _native
    from paper_2209_02882_b200.selector import _first_p
    cases = ((G.chung_lu(232965, 3_000_000, seed=4, device="cuda"), 256),
             (G.rmat(18, 4, seed=5, device="cuda"), 512))
    for g, n in cases:
        a = _device(g)
        rp = a.row_ptr.cpu().numpy().astype(np.int64)
        b = torch.rand((a.num_cols, n), device="cuda") * 2 - 1
        want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(),
                               a.vals.cpu().numpy(), b.cpu().numpy(), n)
        c = torch.empty((a.num_rows, n), device="cuda")
        for text in ("nnz:512,col:4,r:1", "nnz:64,col:2,r:1"):
            p = _first_p(text, n)
            k = lower(algorithm_template(parse_point(text), KernelConfig(n=n, p=p)),
                      _Rp(a.num_rows, a.num_cols, rp), compute_starts=False)
            aux = prepare_aux(k, a)
            wb = {}
            for v in (1, 10):
                for acc in (False, True):
                    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
                    c.zero_() if acc else c.fill_(float("nan"))
                    spmm(k, a, b, c, aux=aux, hw_variant=v, writebacks=cnt, accumulate=acc)
                    assert oracle.max_rel_error(c.cpu().numpy(), want) <= TOL, (n, text, v, acc)
                    wb[v, acc] = int(cnt.item())
            assert wb[1, False] == wb[10, False] and wb[1, True] == wb[10, True], (n, text, wb)
    g = G.rmat(16, 8, seed=2, device="cuda")
    a = _device(g)
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    k = lower(algorithm_template(parse_point("nnz:512,col:4,r:1"), KernelConfig(n=128, p=1024)),
              _Rp(a.num_rows, a.num_cols, rp), compute_starts=False)
    with pytest.raises(_native.SgapError):  # B = 32 MB: fits the L2, no panels
        spmm(k, a, torch.rand((a.num_cols, 128), device="cuda"),
             torch.empty((a.num_rows, 128), device="cuda"), aux=prepare_aux(k, a), hw_variant=10)


def test_cuda_graph_replay_matches_direct_calls():
    """SpmmGraph: a planned call captured once and replayed (new values and
    B written in place between replays) gives the direct call's results for
    the EB walk (zero-fill + walk + long-row fold) and an RB walk."""
    from paper_2209_02882_b200.device import SpmmGraph
    g = G.rmat(16, 16, seed=8, device="cuda")
    a = _device(g)
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    n = 64
    b = torch.rand((a.num_cols, n), device="cuda") * 2 - 1
    c = torch.empty((a.num_rows, n), device="cuda")
    for text, p, v in (("nnz:256,col:4,r:1", 256, 1), ("row:2,col:2,r:1", 256, 4)):
        k = lower(algorithm_template(parse_point(text), KernelConfig(n=n, p=p)),
                  _Rp(a.num_rows, a.num_cols, rp), compute_starts=False)
        gr = SpmmGraph(k, a, b, c, hw_variant=v)
        for step in range(3):
            a.vals.mul_(-1.0 if step % 2 else 0.5)   # new values, same structure
            b.add_(0.25)
            c.fill_(float("nan"))
            gr.replay()
            torch.cuda.synchronize()
            want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(),
                                   a.vals.cpu().numpy(), b.cpu().numpy(), n)
            assert oracle.max_rel_error(c.cpu().numpy(), want) <= TOL, (text, step)
