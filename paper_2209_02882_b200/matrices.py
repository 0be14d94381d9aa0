"""Host-side operand containers, mirroring ``spmmlab.matrices``.

Reference: ``/root/reference/pkg/src/spmmlab/matrices.py``
  CsrMatrix      38-86   (int64 row_ptr/col_idx, float64 vals, invariants)
  DenseMatrix    89-121  (flat row-major float64, index i*num_cols + k)
  _coo_to_csr    124-141 (duplicates combined by summation)
  random_csr     220-233 (seeded; bit-identical generator reproduced here)
  random_dense   236-238

Differences that matter for the B200 path: the invariant checks are
vectorised (the reference walks rows in Python, ~8 us/row), and both classes
can hand their arrays to the device in the layout the kernels use (int32
indices, float32 or float64 values) through ``paper_2209_02882_b200.device``.
There is deliberately no host SpMM here: the product computes on the GPU only.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["CsrMatrix", "DenseMatrix", "MatrixFormatError", "coo_to_csr", "load_matrix_market",
           "loads_matrix_market", "random_csr", "random_dense"]


class MatrixFormatError(ValueError):
    """Malformed Matrix Market input; ``line`` is 1-based (matrices.py:28-36)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(f"line {line}: {message}" if line is not None else message)


def _check_csr(num_rows, num_cols, row_ptr, col_idx, vals):
    if num_rows < 0 or num_cols < 0:
        raise ValueError("matrix dimensions must be non-negative")
    if row_ptr.shape != (num_rows + 1,):
        raise ValueError("row_ptr must have num_rows + 1 entries")
    if row_ptr[0] != 0 or row_ptr[-1] != vals.shape[0]:
        raise ValueError("row_ptr must start at 0 and end at nnz")
    if row_ptr.shape[0] > 1 and np.any(row_ptr[1:] < row_ptr[:-1]):
        raise ValueError("row_ptr must be non-decreasing")
    if col_idx.shape != vals.shape:
        raise ValueError("col_idx and vals must have equal length")
    nnz = vals.shape[0]
    if nnz == 0:
        return
    if col_idx.min() < 0 or col_idx.max() >= num_cols:
        raise ValueError("column index out of range")
    # strictly increasing columns inside every row: every adjacent pair that
    # does not straddle a row start must increase
    step_ok = col_idx[1:] > col_idx[:-1]
    starts = row_ptr[1:-1]
    starts = starts[(starts > 0) & (starts < nnz)]
    crossing = np.zeros(nnz - 1, dtype=bool)
    crossing[starts - 1] = True
    bad = np.flatnonzero(~(step_ok | crossing))
    if bad.size:
        row = int(np.searchsorted(row_ptr, bad[0], side="right") - 1)
        raise ValueError(f"columns in row {row} must be strictly increasing")


@dataclass(frozen=True)
class CsrMatrix:
    """Sparse A in CSR (reference layout: int64 indices, float64 values)."""

    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray

    def __post_init__(self):
        rp = np.asarray(self.row_ptr, dtype=np.int64)
        ci = np.asarray(self.col_idx, dtype=np.int64)
        v = np.asarray(self.vals, dtype=np.float64)
        object.__setattr__(self, "row_ptr", rp)
        object.__setattr__(self, "col_idx", ci)
        object.__setattr__(self, "vals", v)
        _check_csr(self.num_rows, self.num_cols, rp, ci, v)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.num_rows, self.num_cols)

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.num_rows, self.num_cols))
        rows = np.repeat(np.arange(self.num_rows), self.row_lengths())
        out[rows, self.col_idx] = self.vals
        return out


@dataclass
class DenseMatrix:
    """Row-major dense B or C over a flat float64 buffer (index i*num_cols+k)."""

    num_rows: int
    num_cols: int
    vals: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self):
        if self.vals is None:
            self.vals = np.zeros(self.num_rows * self.num_cols)
        self.vals = np.asarray(self.vals, dtype=np.float64).reshape(-1)
        if self.vals.shape[0] != self.num_rows * self.num_cols:
            raise ValueError("vals length must equal num_rows * num_cols")

    @classmethod
    def from_2d(cls, array) -> "DenseMatrix":
        grid = np.asarray(array, dtype=np.float64)
        return cls(grid.shape[0], grid.shape[1], grid.reshape(-1).copy())

    def at(self, i: int, k: int) -> float:
        return float(self.vals[i * self.num_cols + k])

    def to_2d(self) -> np.ndarray:
        return self.vals.reshape(self.num_rows, self.num_cols).copy()

    def dump_text(self) -> str:
        grid = self.vals.reshape(self.num_rows, self.num_cols)
        body = [" ".join(repr(float(x)) for x in row) for row in grid]
        return "\n".join([f"{self.num_rows} {self.num_cols}", *body]) + "\n"


def coo_to_csr(num_rows: int, num_cols: int, rows, cols, vals, *, check: bool = True) -> CsrMatrix:
    """Sort coordinates row-major, sum duplicates, pack CSR (matrices.py:124-141)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size:
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        first = np.empty(rows.size, dtype=bool)
        first[0] = True
        np.not_equal(rows[1:], rows[:-1], out=first[1:])
        first[1:] |= cols[1:] != cols[:-1]
        heads = np.flatnonzero(first)
        if heads.size != rows.size:
            vals = np.add.reduceat(vals, heads)
            rows, cols = rows[heads], cols[heads]
    counts = np.bincount(rows, minlength=num_rows) if rows.size else np.zeros(num_rows, np.int64)
    row_ptr = np.zeros(num_rows + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    if not check:
        m = object.__new__(CsrMatrix)
        for name, value in (("num_rows", num_rows), ("num_cols", num_cols), ("row_ptr", row_ptr),
                            ("col_idx", cols), ("vals", vals)):
            object.__setattr__(m, name, value)
        return m
    return CsrMatrix(num_rows, num_cols, row_ptr, cols, vals)


def _mm_header(lines):
    """Validate banner + size line; returns (rows, cols, nnz, symmetric, first
    entry line index) -- matrices.py:144-186 semantics and line numbers."""
    if not lines:
        raise MatrixFormatError("empty file", 1)
    banner = lines[0].split()
    if len(banner) < 5 or banner[0] != "%%MatrixMarket":
        raise MatrixFormatError("expected '%%MatrixMarket' banner", 1)
    obj, fmt, field, sym = (t.lower() for t in banner[1:5])
    if obj != "matrix" or fmt != "coordinate":
        raise MatrixFormatError(f"unsupported object/format '{obj} {fmt}'", 1)
    if field != "real":
        raise MatrixFormatError(f"unsupported field '{field}' (only real)", 1)
    if sym not in ("general", "symmetric"):
        raise MatrixFormatError(f"unsupported symmetry '{sym}'", 1)
    idx = 1
    while idx < len(lines) and (not lines[idx].strip() or lines[idx].lstrip().startswith("%")):
        idx += 1
    if idx >= len(lines):
        raise MatrixFormatError("missing size line", idx + 1)
    parts = lines[idx].split()
    if len(parts) != 3:
        raise MatrixFormatError("size line must be 'rows cols nnz'", idx + 1)
    try:
        rows, cols, nnz = (int(x) for x in parts)
    except ValueError:
        raise MatrixFormatError("size line must contain integers", idx + 1) from None
    if rows < 0 or cols < 0 or nnz < 0:
        raise MatrixFormatError("size values must be non-negative", idx + 1)
    return rows, cols, nnz, sym == "symmetric", idx + 1


def _mm_entries_checked(lines, start, rows, cols, nnz):
    """Line-by-line entry validation, used to report the exact bad line."""
    r_out, c_out, v_out = [], [], []
    for ln in range(start, len(lines)):
        text = lines[ln].strip()
        if not text or text.startswith("%"):
            continue
        parts = text.split()
        if len(parts) != 3:
            raise MatrixFormatError("entry must be 'row col value'", ln + 1)
        try:
            r, c, v = int(parts[0]), int(parts[1]), float(parts[2])
        except ValueError:
            raise MatrixFormatError(f"non-numeric entry {parts!r}", ln + 1) from None
        if not (1 <= r <= rows and 1 <= c <= cols):
            raise MatrixFormatError(f"coordinate ({r}, {c}) outside {rows}x{cols}", ln + 1)
        r_out.append(r - 1)
        c_out.append(c - 1)
        v_out.append(v)
        if len(r_out) > nnz:
            raise MatrixFormatError("more entries than declared", ln + 1)
    if len(r_out) != nnz:
        raise MatrixFormatError(f"declared {nnz} entries but found {len(r_out)}", len(lines) + 1)
    return np.array(r_out, np.int64), np.array(c_out, np.int64), np.array(v_out, np.float64)


def loads_matrix_market(text: str) -> CsrMatrix:
    """Coordinate Matrix Market (real, general|symmetric) -> CSR, duplicates
    summed, symmetric off-diagonals mirrored (matrices.py:144-212).  Entry
    lines are converted with one vectorised numpy pass; any malformed input
    falls back to the line-by-line check for the exact error line."""
    lines = text.splitlines()
    rows, cols, nnz, symmetric, start = _mm_header(lines)
    body = [ln for ln in lines[start:] if ln.strip() and not ln.lstrip().startswith("%")]
    try:
        tok = np.array(" ".join(body).split(), dtype=object)
        if tok.size != 3 * nnz:
            raise ValueError
        tok = tok.reshape(-1, 3)
        r = tok[:, 0].astype(np.int64) - 1
        c = tok[:, 1].astype(np.int64) - 1
        v = tok[:, 2].astype(np.float64)
        if nnz and (r.min() < 0 or r.max() >= rows or c.min() < 0 or c.max() >= cols):
            raise ValueError
    except (ValueError, TypeError):
        r, c, v = _mm_entries_checked(lines, start, rows, cols, nnz)
    if symmetric:
        off = r != c
        # mirrored entry follows its source, as the reference appends it
        order = np.argsort(np.concatenate([np.arange(r.size) * 2, np.flatnonzero(off) * 2 + 1]),
                           kind="stable")
        r, c, v = (np.concatenate([x, y])[order] for x, y in ((r, c[off]), (c, r[off]), (v, v[off])))
    return coo_to_csr(rows, cols, r, c, v)


def load_matrix_market(path) -> CsrMatrix:
    from pathlib import Path

    return loads_matrix_market(Path(path).read_text())


def random_csr(num_rows: int, num_cols: int, density: float, seed: int) -> CsrMatrix:
    """Seeded uniform-random CSR; bit-identical to the reference generator
    (same ``default_rng`` draw sequence: distinct flat coordinates, then
    U[-1, 1) values)."""
    if not 0.0 <= density <= 1.0:
        raise ValueError("density must be within [0, 1]")
    total = num_rows * num_cols
    nnz = int(round(density * total))
    rng = np.random.default_rng(seed)
    if nnz:
        flat = rng.choice(total, size=nnz, replace=False)
    else:
        flat = np.empty(0, dtype=np.int64)
    vals = rng.uniform(-1.0, 1.0, size=nnz)
    return coo_to_csr(num_rows, num_cols, flat // num_cols, flat % num_cols, vals)


def random_dense(num_rows: int, num_cols: int, seed: int) -> DenseMatrix:
    rng = np.random.default_rng(seed)
    return DenseMatrix(num_rows, num_cols, rng.uniform(-1.0, 1.0, num_rows * num_cols))
