"""Kernel configuration, launch geometry and the block-start partition.

Mirrors the integer half of ``spmmlab.lowering``
(``/root/reference/pkg/src/spmmlab/lowering.py``):

  KernelConfig          84-96    n = dense width, p = thread budget (warp multiple)
  binary_search_before  99-116   largest p in [lo, hi) with a[p] <= target, clamped to lo
  compute_block_starts  119-128  row owning the first position of each chunk
  LoweredKernel         131-139  name / grid_size / block_size / block_starts / family / point
  lower                 649-696  grid = ceil(units / chunk) per decomposition (218-243)

The reference lowers a CIN tree to LLIR for its simulator; the B200 path has
no IR -- a ``LoweredKernel`` here carries the same integers plus the split
factors that select and parameterise the sm_100a kernel.  ``grid_size``,
``block_size`` and ``block_starts`` are bit-exact with the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["KernelConfig", "LoweredKernel", "LoweringError", "binary_search_before",
           "compute_block_starts", "lower"]


class LoweringError(ValueError):
    pass


@dataclass(frozen=True)
class KernelConfig:
    """n: dense column count of B and C; p: parallelism budget the template
    factors are scaled around (a positive multiple of 32, no upper bound)."""

    n: int = 4
    p: int = 256

    def __post_init__(self):
        if self.n < 1:
            raise LoweringError("dense width n must be positive")
        if self.p < 32 or self.p % 32:
            raise LoweringError("parallelism p must be a positive warp multiple")


def binary_search_before(array, lo: int, hi: int, target: int) -> int:
    """Largest p in [lo, hi) with array[p] <= target; lo if none (or empty)."""
    lo, hi = int(lo), int(hi)
    if hi <= lo or array[lo] > target:
        return lo
    while hi - lo > 1:
        mid = (lo + hi) >> 1
        if array[mid] <= target:
            lo = mid
        else:
            hi = mid
    return lo


def compute_block_starts(row_ptr, chunk_size: int, num_blocks: int) -> np.ndarray:
    """int64[num_blocks + 1]: entry b is the last row r (0..num_rows) with
    row_ptr[r] <= b * chunk_size.  Host version; ``sgap_block_starts``
    computes the same array on the device."""
    if chunk_size < 1:
        raise LoweringError("chunk size must be positive")
    targets = np.arange(num_blocks + 1, dtype=np.int64) * int(chunk_size)
    return np.searchsorted(np.asarray(row_ptr, dtype=np.int64), targets, side="right") - 1


@dataclass(frozen=True)
class LoweredKernel:
    """A planned B200 kernel for one (point, config, matrix).

    The first six fields match the reference ``LoweredKernel``; the rest are
    the split factors the device kernel consumes (g, c, r, and ``chunk`` =
    units per logical block)."""

    name: str
    grid_size: int
    block_size: int
    block_starts: np.ndarray | None = None
    family: str | None = None
    point: str | None = None
    n: int = 0
    p: int = 0
    g: int = 1
    c: int = 1
    r: int = 1
    chunk: int = 0
    body: tuple = field(default=(), repr=False)  # no IR: the kernel is native


def lower(template, matrix, *, name: str | None = None, compute_starts: bool = True) -> LoweredKernel:
    """Launch geometry of a template on ``matrix`` (lowering.py:218-243, 649-696).

    Position-chunked families (nnz-*) get ``ceil(nnz / chunk)`` blocks (0 for
    an empty matrix) and a block-start table; row-chunked get
    ``ceil(M / chunk)``; the fused row-column family ``ceil(M * n / chunk)``.
    """
    from .templates import FAMILY_NNZ_MULTIPLE, FAMILY_NNZ_ONE, FAMILY_ROW_MULTIPLE, kernel_name

    fam = template.family
    n = template.config.n
    m = int(matrix.num_rows)
    nnz = int(matrix.row_ptr[-1]) if len(matrix.row_ptr) else 0
    starts = None
    if fam in (FAMILY_NNZ_ONE, FAMILY_NNZ_MULTIPLE):
        grid = -(-nnz // template.chunk) if nnz else 0
        if compute_starts:
            starts = compute_block_starts(matrix.row_ptr, template.chunk, grid)
    elif fam == FAMILY_ROW_MULTIPLE:
        grid = -(-m // template.chunk)
    else:
        grid = -(-(m * n) // template.chunk)
    if template.block_size % 32:
        raise LoweringError(f"thread-block size {template.block_size} is not a warp multiple")
    return LoweredKernel(
        name=name or kernel_name(fam),
        grid_size=grid,
        block_size=template.block_size,
        block_starts=starts,
        family=fam,
        point=str(template.point),
        n=n,
        p=template.config.p,
        g=template.g,
        c=template.c,
        r=template.r,
        chunk=template.chunk,
    )
