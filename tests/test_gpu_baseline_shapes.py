"""Parity at the BASELINE.json shapes the driver benches:

* config 3 (Reddit-shaped, 114.6M nnz) at N = 256,
* config 4 (27-point stencil on 160^3, 109.2M nnz) at N in {16, 64, 256, 512}
  -- the multi-tile lane loops (N/c > 32) run here,
* config 5 (R-MAT scale 24, ~263M nnz, N = 128), one point per family on
  sampled rows (incl. the heaviest),

each through the selector's pick plus one point per family.  The float64
reference product is computed on the device (``sgap_reference_spmm_f64``:
the oracle's exact arithmetic, per-(i, k) ascending-p order, no FMA
contraction) and pinned here to the CPU oracle (``oracle/``) on a row
sample of the same run, so the full-size comparison never needs a host SpMM
of tens of GB.  Bound: 1e-5 in the reference metric (BASELINE.json).

Also: writeback counts (SimMetrics.atomic_ops) for long chunks (g = 64..512)
against the reference simulator's fixtures (tests/golden/sim_long.json)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from paper_2209_02882_b200 import generators as G
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, reference_spmm_f64, spmm
from paper_2209_02882_b200.lowering import KernelConfig, lower
from paper_2209_02882_b200.matrices import CsrMatrix, random_csr, random_dense
from paper_2209_02882_b200.runner import build_kernel
from paper_2209_02882_b200.selector import _first_p, heuristic, matrix_stats
from paper_2209_02882_b200.sim import run
from paper_2209_02882_b200.space import parse_point
from paper_2209_02882_b200.templates import algorithm_template

pytestmark = pytest.mark.gpu

TOL = 1e-5
GOLDEN = Path(__file__).resolve().parent / "golden"


class _Rp:
    def __init__(self, m, k, rp):
        self.num_rows, self.num_cols, self.row_ptr = m, k, rp


def _device(g):
    return DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
                     g.vals.to(torch.float32))


def _rows_sample(rp: np.ndarray, k: int = 3000, heavy: int = 32, seed: int = 0) -> np.ndarray:
    lens = np.diff(rp)
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([np.argsort(-lens)[:heavy],
                                     rng.integers(0, len(lens), k)])).astype(np.int64)


def _pin_device_reference(a: DeviceCsr, b: torch.Tensor, want_dev: torch.Tensor, rows: np.ndarray,
                          n: int) -> None:
    """The device reference equals the CPU oracle (bit for bit) on sampled rows."""
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    lens = np.diff(rp)[rows]
    sub_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    sel = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows]) if lens.sum() else \
        np.zeros(0, np.int64)
    ci = a.col_idx.cpu().numpy()[sel]
    vals = a.vals.cpu().numpy()[sel]
    want = oracle.spmm_f64(sub_rp, ci, vals, b.cpu().numpy(), n)
    got = want_dev[torch.from_numpy(rows).to(want_dev.device)].cpu().numpy()
    assert np.array_equal(got.reshape(-1), want.reshape(-1))


def _device_error(c: torch.Tensor, want: torch.Tensor) -> float:
    worst = 0.0
    step = max(1, (1 << 27) // max(1, c.shape[1]))
    for lo in range(0, c.shape[0], step):  # bounded temporaries
        d = (c[lo:lo + step].double() - want[lo:lo + step]).abs() / (want[lo:lo + step].abs() + 1.0)
        worst = max(worst, float(d.max().item()))
    return worst


def _check_points(g, n: int, points, *, seed: int = 2, label: str = ""):
    """Every (point, p, hw_variant) against the device reference; the
    selector's heuristic pick is added."""
    dev = torch.device("cuda", 0)
    a = _device(g)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    b = torch.rand((g.num_cols, n), generator=gen, device=dev) * 2 - 1
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    want = reference_spmm_f64(a, b, n)
    _pin_device_reference(a, b, want, _rows_sample(rp), n)
    pick = heuristic(matrix_stats(rp, a.num_cols), n)
    items = list(points) + [(pick.point, pick.p, pick.hw_variant)]
    c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
    worst = {}
    for text, p, variant in items:
        p = p if algorithm_template(parse_point(text), KernelConfig(n=n, p=p)) else _first_p(text, n)
        tpl = algorithm_template(parse_point(text), KernelConfig(n=n, p=p))
        assert tpl is not None, text
        k = lower(tpl, _Rp(a.num_rows, a.num_cols, rp), compute_starts=False)
        c.fill_(float("nan"))
        spmm(k, a, b, c, aux=prepare_aux(k, a), hw_variant=variant)
        err = _device_error(c, want)
        worst[(text, p, variant)] = err
        assert err <= TOL, (label, text, p, variant, err)
    print(label, n, worst)
    return worst


def test_config3_n256_every_family():
    """Config 3 (Reddit-shaped) at N = 256: the register, TMA and lane-staged
    EB walks, nnz-one segment + atomic, row-multiple (logical and
    interleaved) and row-reciprocal, plus the selector pick."""
    g = G.config_matrix(3, device="cuda")
    pts = [("nnz:512,col:4,r:1", 256, 1), ("nnz:128,col:4,r:1", 256, 2),
           ("nnz:256,col:4,r:1", 256, 3), ("nnz:1,col:4,r:8", 1024, 0),
           ("nnz:1,col:4,r:1", 256, 0), ("row:4,col:4,r:1", 256, 0),
           ("row:4,col:4,r:1", 256, 2), ("row:1/4,col:4,r:4", 256, 0)]
    _check_points(g, 256, pts, label="config3")


@pytest.mark.parametrize("n", [16, 64, 256, 512])
def test_config4_stencil160_n_sweep(n):
    """Config 4 (27-point stencil on 160^3) across the N sweep: at N/c > 32
    every lane walks several column tiles (tile += W)."""
    g = G.config_matrix(4, device="cuda")
    assert g.nnz == 109_215_352
    c = 4 if n >= 16 else 1
    pts = [(f"nnz:256,col:{c},r:1", 256, 1), (f"nnz:1,col:{c},r:8", 1024, 0),
           (f"row:4,col:{c},r:1", 256, 2), (f"row:1/4,col:{c},r:4", 256, 0)]
    if n // c == 32:
        pts.append((f"row:8,col:{c},r:1", 256, 3))  # warp per row, lane-staged A
    if n // c in (8, 16):
        pts.append((f"row:8,col:{c},r:1", 256, 8))  # shifted blocks, lane groups
    if n // c >= 32:
        pts.append((f"nnz:256,col:{c},r:1", 256, 4))  # lane-staged EB walk
        pts.append((f"row:8,col:{c},r:1", 256, 8))  # shifted 4-row blocks (panels from N=256)
    _check_points(g, n, pts, label="config4")


def test_config5_one_point_per_family_sampled_rows():
    """Config 5 (R-MAT scale 24, 263M nnz, N = 128) at full size: one point
    per family (+ the other EB walks), checked on sampled rows incl. the 64
    heaviest (the full float64 reference would need 17 GB more)."""
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
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    rows = _rows_sample(rp, k=4000, heavy=64, seed=3)
    lens = np.diff(rp)[rows]
    sub_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    sel = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    want = oracle.spmm_f64(sub_rp, a.col_idx.cpu().numpy()[sel], a.vals.cpu().numpy()[sel],
                           b.cpu().numpy(), n)
    rows_d = torch.from_numpy(rows).cuda()
    worst = {}
    for text, p, variant in (("nnz:512,col:4,r:1", 256, 1), ("nnz:512,col:4,r:1", 256, 9),
                             ("nnz:512,col:4,r:1", 256, 5),
                             ("nnz:128,col:4,r:1", 256, 2),
                             ("nnz:256,col:4,r:1", 256, 3), ("nnz:1,col:4,r:8", 1024, 0),
                             ("nnz:1,col:4,r:1", 256, 0), ("row:8,col:4,r:1", 256, 3),
                             ("row:4,col:4,r:1", 256, 0), ("row:1/8,col:4,r:8", 256, 0)):
        tpl = algorithm_template(parse_point(text), KernelConfig(n=n, p=p))
        k = lower(tpl, _Rp(a.num_rows, a.num_cols, rp), compute_starts=False)
        c.fill_(float("nan"))
        spmm(k, a, b, c, aux=prepare_aux(k, a), hw_variant=variant)
        got = c[rows_d].cpu().numpy()
        err = oracle.max_rel_error(got, want)
        worst[(text, variant)] = err
        assert err <= TOL, (text, variant, err)
        assert not torch.isnan(c).any().item(), text
    print("config5", worst)


# --------------------------------------------------------------- long-chunk writebacks

def _sha(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def long_chunk_matrices():
    """Same construction as tests/golden/make_golden.py:long_chunk_matrices
    (pinned by the fixture's hashes)."""
    out = [("random:800x800:0.05:21", random_csr(800, 800, 0.05, seed=21))]
    rng = np.random.default_rng(22)
    m, k = 600, 3000
    lens = np.minimum((rng.pareto(1.2, m) * 8).astype(np.int64), 2500)
    lens[::7] = 0
    lens[3] = 2500
    rp = np.concatenate([[0], np.cumsum(lens)])
    cols = np.concatenate([np.sort(rng.choice(k, int(L), replace=False)) for L in lens if L])
    out.append(("powerlaw:600x3000:22", CsrMatrix(m, k, rp, cols, rng.uniform(-1, 1, rp[-1]))))
    lens = np.zeros(400, dtype=np.int64)
    lens[50:350] = rng.integers(0, 120, 300)
    rp = np.concatenate([[0], np.cumsum(lens)])
    cols = np.concatenate([np.sort(rng.choice(500, int(L), replace=False)) for L in lens if L])
    out.append(("gaps:400x500:22", CsrMatrix(400, 500, rp, cols, rng.uniform(-1, 1, rp[-1]))))
    return out


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("variant", [1, 2])
def test_long_chunk_writebacks_match_simulator(variant, precision):
    """nnz:g for g in 64..512 (the bench's schedules): every EB walk reports
    exactly the reference simulator's atomic_ops (fixtures generated by
    importing spmmlab, tests/golden/make_golden.py --only simlong)."""
    rows = json.loads((GOLDEN / "sim_long.json").read_text())
    mats = dict(long_chunk_matrices())
    n = 8
    cfg = KernelConfig(n=n, p=256)
    checked = 0
    for r in rows:
        mat = mats[r["matrix"]]
        assert _sha(mat.row_ptr) == r["row_ptr_sha"] and _sha(mat.col_idx) == r["col_idx_sha"]
        assert _sha(mat.vals) == r["vals_sha"]
        k = build_kernel(parse_point(r["point"]), cfg, mat)
        assert (k.grid_size, k.block_size) == (r["grid"], r["block"])
        b = random_dense(mat.num_cols, n, seed=5)
        got, m = run(k, mat, b, hw_variant=variant, precision=precision)
        assert m.atomic_ops == r["atomic_ops"], (r["matrix"], r["point"], variant)
        dt = np.float64 if precision == "double" else np.float32
        want = oracle.spmm_f64(np.asarray(mat.row_ptr, np.int32), np.asarray(mat.col_idx, np.int32),
                               np.asarray(mat.vals, dt),
                               np.asarray(b.vals, dt).reshape(mat.num_cols, n), n)
        assert oracle.max_rel_error(got.vals, want) <= (1e-12 if precision == "double" else TOL)
        checked += 1
    assert checked >= 30


# --------------------------------------------------------------- dgSPARSE RB+PR grid

@pytest.mark.parametrize("n", [4, 16, 40, 128])
def test_rbpr_fine_grained_cells(n):
    """The dgSPARSE RB+PR+RM kernel under tuning cells of
    space.enumerate_fine_grained: 2-D blocks narrower than
    a warp, tiles narrower than N, fewer row workers than rows (workerDimR
    scale < 1) and idle extra workers (> 1); float32 within 1e-5 and float64
    within 1e-12 of the oracle, one writeback per output element."""
    from paper_2209_02882_b200.device import spmm_rbpr_grid
    from paper_2209_02882_b200.space import enumerate_fine_grained
    rng = np.random.default_rng(n)
    m, k = 700, 900
    lens = rng.integers(0, 30, m)
    lens[5], lens[9], lens[17] = 850, 0, 880   # rows past 32G: float64 folds
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(k, int(L), replace=False)) for L in lens if L])
    vals = rng.uniform(-1, 1, rp[-1])
    cells = enumerate_fine_grained(n)
    pick = [cells[i] for i in np.random.default_rng(7).choice(len(cells), 24, replace=False)]
    pick += [c for c in cells if (c.group_size, c.block_size, c.tile_size) == (32, 256, 32)]
    for dt, tol in ((torch.float32, TOL), (torch.float64, 1e-12)):
        a = DeviceCsr(m, k, torch.from_numpy(rp.astype(np.int32)).cuda(),
                      torch.from_numpy(cols.astype(np.int32)).cuda(),
                      torch.from_numpy(vals).to(dt).cuda())
        b = (torch.rand((k, n), dtype=torch.float64, device="cuda") * 2 - 1).to(dt)
        want = oracle.spmm_f64(rp.astype(np.int32), cols.astype(np.int32), a.vals.cpu().numpy(),
                               b.cpu().numpy(), n)
        c = torch.empty((m, n), dtype=dt, device="cuda")
        for cell in pick:
            text = f"row:1/{cell.group_size},col:{cell.coarsen_size},r:{cell.group_size}"
            p = _first_p(text, n)
            kk = lower(algorithm_template(parse_point(text), KernelConfig(n=n, p=p)),
                       _Rp(m, k, rp), compute_starts=False)
            wb = torch.zeros(1, dtype=torch.int64, device="cuda")
            c.fill_(float("nan"))
            spmm_rbpr_grid(kk, a, b, c, block=cell.block_size, tile=cell.tile_size,
                           worker_scale=float(cell.worker_scale), writebacks=wb)
            err = oracle.max_rel_error(c.cpu().numpy(), want)
            assert err <= tol, (cell, dt, err)
            assert int(wb.item()) == m * n, cell  # == row-reciprocal's atomic_ops
