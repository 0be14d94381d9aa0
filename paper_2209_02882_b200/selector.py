"""Schedule selection: pick (split, reduction strategy, r, c, p, CTA size).

The reference only enumerates the space (space.py:232-348) and leaves
DA-SpMM's decision tree out of scope; SURVEY 8(a) a20 asks
for a selector driven by nnz/row statistics and N, validated as regret
against an exhaustive sweep.  Two layers:

* ``heuristic(stats, n)`` -- a closed-form rule over the row-length
  statistics (no device work);
* ``autotune(...)`` -- measures candidate kernels on the device operands and
  returns them ranked (the exhaustive sweep when given every candidate).

``tests/test_selector.py`` and ``bench.py --sweep`` report the heuristic's
regret against the sweep.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device import DeviceCsr, panel_lanes, prepare_aux, spmm
from .lowering import KernelConfig, LoweredKernel, lower
from .space import enumerate_space, parse_point
from .templates import algorithm_template

__all__ = ["MatrixStats", "matrix_stats", "Candidate", "candidates", "heuristic", "autotune",
           "plan_for"]


@dataclass(frozen=True)
class MatrixStats:
    num_rows: int
    num_cols: int
    nnz: int
    mean_row: float
    cv_row: float
    max_row: int
    empty_frac: float

    def as_dict(self) -> dict:
        return dict(self.__dict__)


def matrix_stats(row_ptr, num_cols: int) -> MatrixStats:
    rp = np.asarray(row_ptr.cpu() if isinstance(row_ptr, torch.Tensor) else row_ptr, dtype=np.int64)
    lens = np.diff(rp)
    m = lens.shape[0]
    mean = float(lens.mean()) if m else 0.0
    cv = float(lens.std() / mean) if mean > 0 else 0.0
    return MatrixStats(m, int(num_cols), int(rp[-1]), mean, cv, int(lens.max()) if m else 0,
                       float((lens == 0).mean()) if m else 0.0)


@dataclass(frozen=True)
class Candidate:
    point: str
    p: int
    hw_block: int = 0
    hw_variant: int = 0  # nnz-multiple: 1 register / 2 TMA walk; row-multiple: 2 interleaved

    def label(self) -> str:
        return (f"{self.point}@p{self.p}" + (f"/b{self.hw_block}" if self.hw_block else "")
                + (f"/v{self.hw_variant}" if self.hw_variant else ""))


class _RowPtrOnly:
    """Minimal matrix view for host planning (row_ptr + dims)."""

    def __init__(self, num_rows, num_cols, row_ptr):
        self.num_rows, self.num_cols, self.row_ptr = num_rows, num_cols, row_ptr


def plan_for(cand: Candidate, n: int, num_rows: int, num_cols: int, row_ptr_host) -> LoweredKernel | None:
    tpl = algorithm_template(parse_point(cand.point), KernelConfig(n=n, p=cand.p))
    if tpl is None:
        return None
    return lower(tpl, _RowPtrOnly(num_rows, num_cols, row_ptr_host), compute_starts=False)


# The B200 knob grid widens the reference's default g in {2..32}
# (space.py:220) with longer serial chunks, which the EB walk amortises
# best on power-law matrices; the point grammar already admits any g >= 2.
GPU_G_VALUES = (2, 4, 8, 16, 32, 64, 128, 256, 512)
L2_BYTES = 126 << 20  # B200 (cudaDevAttrL2CacheSize: 132,644,864)


def candidates(n: int, p_values=(256, 1024), g_values=GPU_G_VALUES,
               variants: bool = True) -> list[Candidate]:
    """Every templated point at dense width n for each p (deduplicated by
    the kernel it lowers to); nnz-multiple points come with every walk
    (register-staged on row_ptr or on row ids, TMA-staged, lane-staged) and row-multiple points with
    the logical, interleaved and warp-per-row mappings when ``variants``."""
    out, seen = [], set()
    for p in p_values:
        cfg = KernelConfig(n=n, p=p)
        for pt in enumerate_space(g_values=g_values).legal:
            tpl = algorithm_template(pt, cfg)
            if tpl is None:
                continue
            key = (tpl.family, tpl.g, tpl.c, tpl.r, tpl.chunk)
            if key in seen:
                continue
            seen.add(key)
            if variants and tpl.family == "nnz-multiple":
                # 1: register walk tracking rows through row_ptr (DRAM-bound
                # matrices: configs 3/5), 5: the same walk on per-position row
                # ids (latency-bound: config 2), 2: TMA-staged, 3: lane-staged
                # 9: 1 + the plan's cold-column cache hints (B >> L2: config 5)
                # 10: 1 in column panels (B > L2, a panel fits half of it:
                # config 3 at N = 256; refused -- and skipped -- elsewhere)
                vs = (1, 5, 9, 2, 3) if n // tpl.c >= 32 else (1, 5, 9, 2)
                if n // tpl.c > 8:
                    vs += (10,)
                out.extend(Candidate(str(pt), p, 0, v) for v in vs)
            elif variants and tpl.family == "nnz-one":
                # 0: the shuffle segment scan; 1: each segment group walked
                # serially by lanes along the columns (full-row gathers)
                out.extend(Candidate(str(pt), p, 0, v) for v in (0, 1))
            elif variants and tpl.family == "row-multiple" and n // tpl.c <= 256:
                # 6/7: a warp per 4/8-row block walking the union of the
                # block's columns (rows <= 64; stencils / meshes)
                # 4 at N/c = 64, 96, ...: the warp-per-row walk once per
                # 32c-column panel (config 4 at N = 256 / 512)
                L = n // tpl.c
                # 3/4 at N/c = 16 / 8 / 4 / 2: 2 / 4 / 8 / 16 rows per warp
                # (config 4 at N = 64 / 32 / 16)
                # 8 at N/c a multiple of 32: shifted blocks of 4 rows
                # (banded rows share shifted column lists; other blocks fall
                # back to the warp-per-row walk inline)
                vs = ((0, 2, 4, 6, 7, 8) if L == 32 else (0, 2, 4, 8) if L % 32 == 0
                      else (0, 2, 3, 4, 8) if L in (8, 16)
                      else (0, 2, 4) if L in (2, 4)
                      else (0, 2))
                out.extend(Candidate(str(pt), p, 0, v) for v in vs)
            else:
                out.append(Candidate(str(pt), p))
    return out


def _templated(point: str, n: int, p: int) -> bool:
    return algorithm_template(parse_point(point), KernelConfig(n=n, p=p)) is not None


def _first_p(point: str, n: int) -> int | None:
    """256, 1024 or 4096 when templated there, else the smallest warp
    multiple that makes the point's divisibility gates pass."""
    for p in (256, 1024, 4096):
        if _templated(point, n, p):
            return p
    for p in range(32, 32 * 1024, 32):
        if _templated(point, n, p):
            return p
    return None


def _pow2_floor(x: float) -> int:
    out = 1
    while out * 2 <= x:
        out *= 2
    return out


def heuristic(stats: MatrixStats, n: int, esz: int = 4) -> Candidate:
    """Closed-form schedule choice from row statistics and n, fitted to the
    round-1 B200 sweeps (profiles/r01_sweep_*.json, r01_paper_claims.md);
    ``esz`` = bytes per value (8 for float64: vectors of at most 2 values,
    profiles/r02_f64_configs.md):

    * regular rows (cv < 1, max <= 8 x mean):
      - n >= 16: RB + serial, 4 rows per logical thread, interleaved CTA
        mapping, c = 4 (27-pt stencil at N=128);
      - long rows (mean >= 32): RB + parallel group -- 8 lanes over single
        columns for n <= 8, 2 lanes otherwise (uniform 1%: flexible small
        groups beat r=32 at every n);
      - n < 16 and short rows: RB + serial, one lane per row with the widest
        vector (stencil at N=4/8);
    * skewed rows (power law, hub rows): EB + serial walk with the widest
      vector that keeps >= 4 lanes per chunk for small n, chunk g ~ nnz/40k
      clamped to [32, 512] so every warp slot gets several chunks.
    """
    widest = 4 if n % 4 == 0 else (2 if n % 2 == 0 else 1)
    if esz == 8:  # float64: 16-byte vectors are 2 values (config 2/3/4 in
        widest = min(widest, 2)  # float64: col:2 1.4-2.0x faster than col:4)
    col = lambda c: "1" if c == 1 else str(c)  # noqa: E731
    regular = stats.cv_row < 1.0 and stats.max_row <= 8 * max(stats.mean_row, 1.0)
    if regular:
        if stats.mean_row >= 32:
            # long regular rows: a small parallel group; narrow N wants a
            # wider group over single columns (config 1 sweeps: n=4 best
            # row:1/8,col:1,r:8, n=32 row:1/2,col:2,r:2)
            if n <= 8:
                pt = "row:1/8,col:1,r:8"
            elif n <= 32:
                pt = f"row:1/2,col:{col(min(widest, 2))},r:2"
            else:
                pt = f"row:1/2,col:{col(widest)},r:2"
            p = _first_p(pt, n)
            if p is not None:
                return Candidate(pt, p)
        if n >= 16:
            # 8 rows per logical thread from N = 64 (stencil 64^3 N=64, config 4
            # N=128: the round-2 sweeps), 4 below (config 4 N=16)
            pt = f"row:{8 if n >= 64 else 4},col:{col(widest)},r:1"
            p = _first_p(pt, n)
            if p is not None:
                # a warp per row when N/c == 32 (config 4 N=128: 3.35 vs 3.82 ms)
                # and once per 32c-column panel when N/c is a larger multiple
                # of 32 (config 4 N=256 / 512: 6.10 / 12.21 ms vs 7.50 / 15.68
                # for the best full-width schedule, profiles/r02_rb_panels_cfg4.md),
                # and 2 / 4 rows per warp at N/c == 16 / 8 (config 4 N=64 / 32:
                # 1.60 / 0.92 ms vs 1.94 / 1.11 for the logical mapping,
                # profiles/r02_rb_subwarp_cfg4.md), 8 rows per warp at N/c == 4
                # (config 4 N=16: 0.52 vs 0.69 ms for adjacent rows per CTA step)
                # At N/c a multiple of 32 the shifted-block walk (variant 8),
                # which is the warp-per-row walk on blocks whose rows are not
                # shifted copies of each other (config 4 N=128: 2.06 vs 3.07
                # ms, N=256 / 512: 0.67x, profiles/r02_rb_shifted_cfg4.md)
                lanes = n // widest
                if lanes % 32 == 0 or lanes in (8, 16):  # (N=64 / 32: 1.24 / 0.88 vs 1.61 / 0.93 ms)
                    return Candidate(pt, p, 0, 8)
                return Candidate(pt, p, 0, 4 if lanes in (4, 8, 16) else 2)
        pt = f"row:1,col:{col(widest)},r:1"
        return Candidate(pt, _first_p(pt, n) or 256)
    c = widest if n >= 16 else min(widest, max(1, n // 4))
    if n <= 4:
        # narrow B on power-law rows: segment groups of 16, walked serially
        # (nnz-one variant 1; R-MAT s18 N=4 best of the whole sweep)
        pt = f"nnz:1,col:{col(c)},r:16"
        p = _first_p(pt, n)
        if p is not None:
            return Candidate(pt, p, 0, 1)
    # long chunks amortise the walk on wide B; narrow B wants more, shorter
    # chunks (config 2 / Chung-Lu at N = 8: g = 64)
    g = 64 if n <= 16 else max(32, min(512, _pow2_floor(stats.nnz / 40_000)))
    # the register walk's flavour (round-2 interleaved A/B, profiles/r02_ab_*):
    # B far beyond the L2 -> row_ptr tracking + cold-column cache hints
    # (config 5: DRAM-bound, -4.5%); short rows with many empty rows -> the
    # per-position row ids (config 2: every row change of the row_ptr walk
    # waits on row_ptr loads, 56% / 48% empty rows); otherwise row_ptr
    # tracking with the column-pipelined batches (config 3 at N = 64 / 256)
    b_bytes = stats.num_cols * n * esz
    if b_bytes > 1.5 * L2_BYTES and panel_lanes(stats.num_cols, n, c, esz) >= 16:
        # B well beyond the L2 but a column panel of >= 16 tiles fits half of
        # it: walk the panels one at a time (config 3 at N = 256: 0.79x of
        # variant 1, profiles/r02_sweeps/); not for B just above the L2 with
        # narrow panels (hold-out Chung-Lu 300k at N = 128, B = 154 MB,
        # 32-column panels: 1.22x slower than variant 1)
        variant = 10
    elif b_bytes > 16 * L2_BYTES:
        variant = 9
    elif stats.mean_row < 32 and stats.empty_frac > 0.2:
        variant = 5
    elif b_bytes > 1.5 * L2_BYTES:  # the planner builds hints from here (device.py)
        variant = 9                 # (config 3 at N=256: -3.2% vs variant 1)
    else:
        variant = 1
    for gg in (g, 256, 128, 64, 32):
        pt = f"nnz:{gg},col:{col(c)},r:1"
        p = _first_p(pt, n)
        if p is not None:
            return Candidate(pt, p, 0, variant if gg % 4 == 0 else 5)
    pt = f"row:1,col:{col(widest)},r:1"
    return Candidate(pt, _first_p(pt, n) or 256)


def autotune(a: DeviceCsr, b: torch.Tensor, c: torch.Tensor, n: int, cands, *, reps: int = 3,
             row_ptr_host=None, stream=None, max_ms: float | None = None) -> list[tuple[Candidate, float]]:
    """Time each candidate (zero-fill included for atomic families); returns
    [(candidate, best ms)] fastest first.  Candidates slower than ``max_ms``
    on their first run are not repeated."""
    rp = row_ptr_host if row_ptr_host is not None else a.row_ptr.cpu().numpy()
    stream = stream or torch.cuda.current_stream()
    results = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for cand in cands:
        k = plan_for(cand, n, a.num_rows, a.num_cols, rp)
        if k is None:
            continue
        aux = prepare_aux(k, a, stream=stream)
        try:
            spmm(k, a, b, c, aux=aux, hw_block=cand.hw_block, hw_variant=cand.hw_variant,
                 stream=stream)  # warm
        except _native.SgapError as e:
            if e.status != _native.ERR_ARG:  # only "variant not applicable" is skipped
                raise
            continue
        best = float("inf")
        for i in range(reps):
            e0.record(stream)
            spmm(k, a, b, c, aux=aux, hw_block=cand.hw_block, hw_variant=cand.hw_variant,
                 stream=stream)
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
            if max_ms is not None and best > max_ms:
                break
        results.append((cand, best))
    results.sort(key=lambda t: t[1])
    return results


def refine(a: DeviceCsr, b: torch.Tensor, c: torch.Tensor, n: int, ranked, *, top: int = 6,
           rounds: int = 4, reps: int = 3, row_ptr_host=None, stream=None):
    """Re-time the ``top`` candidates of an ``autotune`` ranking in
    interleaved rounds (median of ``reps`` launches per round, median over
    rounds), so clock and power drift during the sweep cannot pick a
    candidate that is only a few percent ahead by luck (config 5's walks
    differ by 3-5%).  Returns [(candidate, ms)] fastest first."""
    import statistics
    rp = row_ptr_host if row_ptr_host is not None else a.row_ptr.cpu().numpy()
    stream = stream or torch.cuda.current_stream()
    arms = []
    for cand, _ in ranked[:top]:
        k = plan_for(cand, n, a.num_rows, a.num_cols, rp)
        arms.append((cand, k, prepare_aux(k, a, stream=stream)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = {id(cd): [] for cd, _, _ in arms}
    for _ in range(rounds):
        for cand, k, aux in arms:
            ts = []
            for _ in range(reps):
                e0.record(stream)
                spmm(k, a, b, c, aux=aux, hw_block=cand.hw_block, hw_variant=cand.hw_variant,
                     stream=stream)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            times[id(cand)].append(statistics.median(ts))
    out = [(cand, statistics.median(times[id(cand)])) for cand, _, _ in arms]
    out.sort(key=lambda t: t[1])
    return out
