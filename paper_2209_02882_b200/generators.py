"""Seeded synthetic matrices for the BASELINE.json workloads.

The reference only has ``random_csr`` (matrices.py:220-233), which draws
``rng.choice(M*K)`` densely and cannot produce configs 2-5, so
the larger shapes are generated here:

  config 1  random_csr(4096, 4096, 0.01, seed=1)      (matrices.random_csr, bit-exact)
  config 2  R-MAT scale 20, edge factor 16            rmat(20, 16)
  config 3  Reddit-shaped 232,965 rows, ~114.6M nnz    chung_lu(232965, 114.6e6)
  config 4  27-point stencil on 160^3                  stencil27(160)
  config 5  R-MAT scale 24, edge factor 16            rmat(24, 16)

Values are U[-1, 1).  Duplicate coordinates are summed (the reference's
``_coo_to_csr`` rule).  Generation is vectorised with torch on whichever
device is given (the GPU for the big configs: tens of seconds on the host
become milliseconds); it is input preparation, not part of the timed SpMM.
Outputs are (row_ptr int64, col_idx int64, vals float64) tensors on that
device, or a ``CsrMatrix`` via ``to_csr``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .matrices import CsrMatrix

__all__ = ["GeneratedCsr", "rmat", "stencil27", "chung_lu", "uniform_random", "to_csr", "config_matrix"]

GRAPH500 = (0.57, 0.19, 0.19, 0.05)


@dataclass
class GeneratedCsr:
    num_rows: int
    num_cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    vals: torch.Tensor
    label: str

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())


def _pack(num_rows: int, num_cols: int, rows: torch.Tensor, cols: torch.Tensor,
          vals: torch.Tensor, label: str) -> GeneratedCsr:
    """Row-major sort, duplicate coordinates summed, CSR row pointer."""
    key = rows.to(torch.int64) * num_cols + cols.to(torch.int64)
    key, order = torch.sort(key, stable=True)
    vals = vals[order]
    uniq, inverse = torch.unique_consecutive(key, return_inverse=True)
    if uniq.numel() != key.numel():
        summed = torch.zeros(uniq.numel(), dtype=vals.dtype, device=vals.device)
        summed.index_add_(0, inverse, vals)
        vals = summed
    rows = torch.div(uniq, num_cols, rounding_mode="floor")
    cols = uniq - rows * num_cols
    counts = torch.bincount(rows, minlength=num_rows)
    row_ptr = torch.zeros(num_rows + 1, dtype=torch.int64, device=rows.device)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    return GeneratedCsr(num_rows, num_cols, row_ptr, cols, vals, label)


def _uniform(n: int, gen: torch.Generator, device) -> torch.Tensor:
    return torch.rand(n, generator=gen, dtype=torch.float64, device=device) * 2.0 - 1.0


def rmat(scale: int, edge_factor: int = 16, *, seed: int = 1, params=GRAPH500,
         permute: bool = True, device="cpu") -> GeneratedCsr:
    """Graph500 R-MAT: 2^scale vertices, edge_factor * 2^scale directed edges,
    quadrant probabilities (a, b, c, d); no self-loop removal; duplicates
    summed; a seeded vertex permutation applied to rows and columns unless
    ``permute=False`` (the unpermuted stress case)."""
    a, b, c, _ = params
    n = 1 << scale
    m = edge_factor * n
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    rows = torch.zeros(m, dtype=torch.int64, device=device)
    cols = torch.zeros(m, dtype=torch.int64, device=device)
    for level in range(scale):
        u = torch.rand(m, generator=gen, dtype=torch.float32, device=device)
        row_bit = u >= (a + b)
        col_bit = ((u >= a) & (u < a + b)) | (u >= a + b + c)
        bit = 1 << (scale - 1 - level)
        rows += row_bit.to(torch.int64) * bit
        cols += col_bit.to(torch.int64) * bit
        del u, row_bit, col_bit
    if permute:
        perm = torch.randperm(n, generator=gen, device=device)
        rows = perm[rows]
        cols = perm[cols]
    vals = _uniform(m, gen, device)
    tag = "" if permute else ",unpermuted"
    return _pack(n, n, rows, cols, vals, f"rmat:scale={scale},ef={edge_factor},seed={seed}{tag}")


def stencil27(side: int, *, seed: int = 1, device="cpu") -> GeneratedCsr:
    """27-point stencil on a side^3 grid (x fastest): row (x,y,z) couples to
    every in-bounds (x+dx, y+dy, z+dz), |d*| <= 1.  nnz = (3*side - 2)^3."""
    n = side ** 3
    idx = torch.arange(n, dtype=torch.int64, device=device)
    x = idx % side
    y = (idx // side) % side
    z = idx // (side * side)
    cols = torch.empty((n, 27), dtype=torch.int64, device=device)
    valid = torch.empty((n, 27), dtype=torch.bool, device=device)
    j = 0
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):  # ascending linear offset -> ascending column
                ok = ((x + dx >= 0) & (x + dx < side) & (y + dy >= 0) & (y + dy < side)
                      & (z + dz >= 0) & (z + dz < side))
                cols[:, j] = idx + dx + dy * side + dz * side * side
                valid[:, j] = ok
                j += 1
    counts = valid.sum(1)
    col_idx = cols[valid]
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    vals = _uniform(col_idx.numel(), gen, device)
    return GeneratedCsr(n, n, row_ptr, col_idx, vals, f"stencil27:side={side},seed={seed}")


def chung_lu(num_rows: int, target_nnz: float, *, seed: int = 1, alpha: float = 1.6,
             device="cpu") -> GeneratedCsr:
    """Symmetric Chung-Lu graph with a heavy-tailed (Pareto, tail index
    ``alpha``) expected-degree sequence, sized so the deduplicated nnz lands
    near ``target_nnz`` -- a seeded stand-in for the Reddit GNN adjacency
    (232,965 nodes, ~114.6M nnz); the real dataset is not available offline."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    u = torch.rand(num_rows, generator=gen, dtype=torch.float64, device=device)
    w = (1.0 - u).pow(-1.0 / alpha)
    w = torch.clamp(w / w.mean() * (target_nnz / num_rows), max=float(num_rows) * 0.5)
    probs = (w / w.sum()).to(torch.float32)
    draws = int(target_nnz / 2)
    out = None
    for _ in range(4):  # grow the draw count until dedup lands near the target
        src = torch.multinomial(probs, draws, replacement=True, generator=gen)
        dst = torch.multinomial(probs, draws, replacement=True, generator=gen)
        rows = torch.cat([src, dst])
        cols = torch.cat([dst, src])
        vals = _uniform(rows.numel(), gen, device)
        out = _pack(num_rows, num_rows, rows, cols, vals,
                    f"chung_lu:rows={num_rows},target={int(target_nnz)},seed={seed}")
        if out.nnz >= 0.97 * target_nnz:
            break
        draws = int(draws * min(2.0, target_nnz / max(out.nnz, 1)))
        del src, dst, rows, cols, vals
    return out


def uniform_random(num_rows: int, num_cols: int, nnz_per_row: float, *, seed: int = 1,
                   device="cpu") -> GeneratedCsr:
    """Uniform random coordinates with replacement (duplicates summed);
    for large uniform matrices where random_csr's dense draw is infeasible."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    m = int(num_rows * nnz_per_row)
    rows = torch.randint(0, num_rows, (m,), generator=gen, device=device)
    cols = torch.randint(0, num_cols, (m,), generator=gen, device=device)
    return _pack(num_rows, num_cols, rows, cols, _uniform(m, gen, device),
                 f"uniform:{num_rows}x{num_cols},nnz/row={nnz_per_row},seed={seed}")


def to_csr(g: GeneratedCsr, *, check: bool = False) -> CsrMatrix:
    """Host CsrMatrix (int64/float64) of a generated matrix."""
    rp = g.row_ptr.cpu().numpy()
    ci = g.col_idx.cpu().numpy()
    v = g.vals.cpu().numpy()
    if check:
        return CsrMatrix(g.num_rows, g.num_cols, rp, ci, v)
    m = object.__new__(CsrMatrix)
    for name, value in (("num_rows", g.num_rows), ("num_cols", g.num_cols), ("row_ptr", rp),
                        ("col_idx", ci), ("vals", v)):
        object.__setattr__(m, name, value)
    return m


def config_matrix(cfg: int, *, device="cpu", seed: int = 1) -> GeneratedCsr:
    """The sparse operand of BASELINE.json config ``cfg`` (1-5)."""
    if cfg == 1:
        from .matrices import random_csr
        a = random_csr(4096, 4096, 0.01, seed=seed)
        t = lambda x: torch.from_numpy(np.asarray(x)).to(device)  # noqa: E731
        return GeneratedCsr(4096, 4096, t(a.row_ptr), t(a.col_idx), t(a.vals),
                            f"random_csr:4096x4096:0.01:{seed}")
    if cfg == 2:
        return rmat(20, 16, seed=seed, device=device)
    if cfg == 3:
        return chung_lu(232_965, 114.6e6, seed=seed, device=device)
    if cfg == 4:
        return stencil27(160, seed=seed, device=device)
    if cfg == 5:
        return rmat(24, 16, seed=seed, device=device)
    raise ValueError(f"unknown config {cfg}")
