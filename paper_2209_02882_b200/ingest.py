"""Matrix Market -> device CSR (device-side ingest).

``load_matrix_market_device(text)`` is ``matrices.loads_matrix_market``
(reference ``matrices.py:144-212`` + ``_coo_to_csr`` ``124-141``) with the
per-entry work on the GPU:

* host: the banner and size line (``matrices._mm_header``, same errors);
* device (libsgap.so): index the body's lines, tokenise and convert every
  entry line with one thread per line (``sgap_mm_parse``), expand symmetric
  entries in the reference's append order, stable-sort the COO keys, sum
  duplicate runs in np.add.reduceat order (``sgap_mm_sum_runs``) and build
  row_ptr;
* host again, only where needed: lines whose tokens fall outside the strict
  device grammar (underscores, inf/nan) are converted with Python's own
  int()/float(); plain decimals the device cannot convert exactly (> 19
  significant digits, subnormal or overflowing: Clinger's fast path and
  Eisel-Lemire cover the rest) in one numpy batch,
  and the first bad line (if any) is re-checked in Python for the reference's
  exact message and line number.

The result is bit-identical to the host parser (values, indices, errors);
tests/test_gpu_ingest.py compares the two.  torch provides the sort, scans
and compactions (library primitives, like cub); the parsing and the
duplicate-summation order are ours.
"""

from __future__ import annotations

import ctypes
import re
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device import DeviceCsr
from .matrices import MatrixFormatError, _mm_header, loads_matrix_market

__all__ = ["DeviceCoo", "load_matrix_market_device"]

SKIP, OK, FIELDS, NONNUM, RANGE, HOST, FLOAT = range(7)


@dataclass
class DeviceCoo:
    """Device CSR as the reference's CsrMatrix holds it: int64 indices,
    float64 values (``to_csr`` narrows to the SpMM layout)."""

    num_rows: int
    num_cols: int
    row_ptr: torch.Tensor  # int64 [num_rows + 1]
    col_idx: torch.Tensor  # int64 [nnz]
    vals: torch.Tensor     # float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    def to_csr(self, dtype=torch.float32) -> DeviceCsr:
        if self.nnz >= 2**31 or self.num_rows >= 2**31 - 1:
            raise ValueError("the SpMM engine takes int32 indices")
        return DeviceCsr(self.num_rows, self.num_cols, self.row_ptr.to(torch.int32),
                         self.col_idx.to(torch.int32), self.vals.to(dtype))


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _check_line(text: str, rows: int, cols: int):
    """The reference's per-line logic (matrices.py:190-204) for one line:
    (status, r, c, v, message)."""
    s = text.strip()
    if not s or s.startswith("%"):
        return SKIP, 0, 0, 0.0, None
    parts = s.split()
    if len(parts) != 3:
        return FIELDS, 0, 0, 0.0, "entry must be 'row col value'"
    try:
        r, c, v = int(parts[0]), int(parts[1]), float(parts[2])
    except ValueError:
        return NONNUM, 0, 0, 0.0, f"non-numeric entry {parts!r}"
    if not (1 <= r <= rows and 1 <= c <= cols):
        return RANGE, 0, 0, 0.0, f"coordinate ({r}, {c}) outside {rows}x{cols}"
    return OK, r - 1, c - 1, v, None


def _host_csr(text: str, device) -> DeviceCoo:
    m = loads_matrix_market(text)
    dev = torch.device(device)
    return DeviceCoo(m.num_rows, m.num_cols, torch.as_tensor(m.row_ptr, device=dev),
                     torch.as_tensor(m.col_idx, dtype=torch.int64, device=dev),
                     torch.as_tensor(m.vals, dtype=torch.float64, device=dev))


def load_matrix_market_device(text: str | bytes, device="cuda", stats: dict | None = None) -> DeviceCoo:
    """Coordinate Matrix Market (real, general|symmetric) -> CSR on ``device``;
    same result and errors as ``matrices.loads_matrix_market``.  ``stats``
    (optional dict) receives how many body lines were parsed and how many
    values / lines the host had to convert or judge."""
    if isinstance(text, (bytes, bytearray)):
        text = bytes(text).decode()
    dev = torch.device(device)
    L = _native.lib()
    # header on the host: the banner, comments and the size line
    head_lines, pos = [], 0
    while pos < len(text):  # text.splitlines() up to the size line
        nl = text.find("\n", pos)
        line = text[pos:] if nl < 0 else text[pos:nl]
        head_lines.append(line)
        pos = len(text) if nl < 0 else nl + 1
        s = line.strip()
        if len(head_lines) > 1 and s and not s.startswith("%"):
            break
    if re.search(r"\r(?!\n)|[\x0b\x0c\x1c\x1d\x1e]", text[:pos]) or not text.isascii():
        return _host_csr(text, dev)  # separators a '\n' scan does not see: the host parser
    rows, cols, nnz, symmetric, start = _mm_header(head_lines)
    body = text[pos:].encode()
    first_line = start  # 0-based index of the body's first line in text.splitlines()
    if len(body) >= 2**31:
        return _host_csr(text, dev)  # the line index uses 32-bit selection
    if rows >= 2**31 or cols >= 2**31:
        return _host_csr(text, dev)  # COO sort keys pack (row << 32 | col)
    st = torch.cuda.current_stream(dev).cuda_stream
    d_text = torch.frombuffer(bytearray(body), dtype=torch.uint8).to(dev) if body else \
        torch.empty(0, dtype=torch.uint8, device=dev)
    flags = torch.empty(len(body), dtype=torch.uint8, device=dev)
    special = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.check(L.sgap_mm_line_flags(_ptr(d_text), len(body), _ptr(flags), _ptr(special), st),
                  "sgap_mm_line_flags")
    if int(special.item()):
        return _host_csr(text, dev)
    starts = torch.nonzero(flags, as_tuple=True)[0].to(torch.int64) if len(body) else \
        torch.empty(0, dtype=torch.int64, device=dev)
    nlines = int(starts.numel())
    status = torch.empty(nlines, dtype=torch.uint8, device=dev)
    r = torch.empty(nlines, dtype=torch.int64, device=dev)
    c = torch.empty(nlines, dtype=torch.int64, device=dev)
    v = torch.empty(nlines, dtype=torch.float64, device=dev)
    tok_off = torch.empty(nlines, dtype=torch.int64, device=dev)
    tok_len = torch.empty(nlines, dtype=torch.int32, device=dev)
    _native.check(L.sgap_mm_parse(_ptr(d_text), len(body), _ptr(starts), nlines, rows, cols,
                                  _ptr(status), _ptr(r), _ptr(c), _ptr(v), _ptr(tok_off),
                                  _ptr(tok_len), st), "sgap_mm_parse")
    # plain decimals off the exact fast path (e.g. 17-digit repr values):
    # converted in one batch by numpy's bytes -> float64 (correctly rounded,
    # bit-identical to float()), gathered from the host copy of the text
    fl_idx = torch.nonzero(status == FLOAT, as_tuple=True)[0]
    if stats is not None:
        stats.update(lines=nlines, host_floats=int(fl_idx.numel()),
                     host_lines=int((status == HOST).sum().item()))
    if fl_idx.numel():
        off = tok_off[fl_idx].cpu().numpy()
        ln = tok_len[fl_idx].cpu().numpy().astype(np.int64)
        src = np.frombuffer(body, dtype=np.uint8)
        seg = ln + 1  # token + one separating space
        gather = np.repeat(off - np.concatenate([[0], np.cumsum(seg)[:-1]]), seg) + np.arange(seg.sum())
        buf = src[np.minimum(gather, len(src) - 1)].copy()
        buf[np.cumsum(seg) - 1] = ord(" ")
        vals = np.array(buf.tobytes().split(), dtype=np.float64)
        v[fl_idx] = torch.as_tensor(vals, device=dev)
        status[fl_idx] = OK
    # lines only Python can judge
    host_idx = torch.nonzero(status == HOST, as_tuple=True)[0].cpu().numpy()
    if host_idx.size:
        sts = starts.cpu().numpy()
        fix_s, fix_r, fix_c, fix_v = [], [], [], []
        for li in host_idx:
            b0 = int(sts[li])
            b1 = int(sts[li + 1]) - 1 if li + 1 < nlines else len(body)
            stt, rr, cc, vv, _ = _check_line(body[b0:b1].decode(), rows, cols)
            fix_s.append(stt), fix_r.append(rr), fix_c.append(cc), fix_v.append(vv)
        hi = torch.as_tensor(host_idx, dtype=torch.int64, device=dev)
        status[hi] = torch.as_tensor(fix_s, dtype=torch.uint8, device=dev)
        r[hi] = torch.as_tensor(fix_r, dtype=torch.int64, device=dev)
        c[hi] = torch.as_tensor(fix_c, dtype=torch.int64, device=dev)
        v[hi] = torch.as_tensor(fix_v, dtype=torch.float64, device=dev)
    # the first error in file order: a bad line, or the (nnz+1)-th entry
    ok = status == OK
    bad = (status == FIELDS) | (status == NONNUM) | (status == RANGE)
    seen = torch.cumsum(ok.to(torch.int64), 0) if nlines else ok.to(torch.int64)
    first_bad = int(torch.nonzero(bad, as_tuple=True)[0][:1].cpu().sum()) if bool(bad.any()) else nlines
    excess = torch.nonzero(ok & (seen > nnz), as_tuple=True)[0][:1]
    first_excess = int(excess.cpu().sum()) if excess.numel() else nlines
    if first_bad < nlines or first_excess < nlines:
        li = min(first_bad, first_excess)
        lineno = first_line + li + 1
        if li == first_bad:
            b0 = int(starts[li].item())
            b1 = int(starts[li + 1].item()) - 1 if li + 1 < nlines else len(body)
            raise MatrixFormatError(_check_line(body[b0:b1].decode(), rows, cols)[4], lineno)
        raise MatrixFormatError("more entries than declared", lineno)
    found = int(seen[-1].item()) if nlines else 0
    if found != nnz:
        total_lines = first_line + nlines
        raise MatrixFormatError(f"declared {nnz} entries but found {found}", total_lines + 1)
    # COO in append order, stable sort by (row, col), duplicate sums
    mult = ok.to(torch.int64)
    if symmetric:
        mult = mult + (ok & (r != c)).to(torch.int64)
    total = int(mult.sum().item())
    pos_t = torch.cumsum(mult, 0) - mult
    key = torch.empty(total, dtype=torch.int64, device=dev)
    val = torch.empty(total, dtype=torch.float64, device=dev)
    _native.check(L.sgap_mm_expand(nlines, _ptr(status), _ptr(r), _ptr(c), _ptr(v), _ptr(pos_t),
                                   1 if symmetric else 0, _ptr(key), _ptr(val), st), "sgap_mm_expand")
    key_s, order = torch.sort(key, stable=True)
    val_s = val[order]
    if total:
        head = torch.ones(total, dtype=torch.bool, device=dev)
        head[1:] = key_s[1:] != key_s[:-1]
        run_start = torch.nonzero(head, as_tuple=True)[0].to(torch.int64)
    else:
        run_start = torch.empty(0, dtype=torch.int64, device=dev)
    nruns = int(run_start.numel())
    out_r = torch.empty(nruns, dtype=torch.int64, device=dev)
    out_c = torch.empty(nruns, dtype=torch.int64, device=dev)
    out_v = torch.empty(nruns, dtype=torch.float64, device=dev)
    _native.check(L.sgap_mm_sum_runs(total, _ptr(key_s), _ptr(val_s), _ptr(run_start), nruns,
                                     _ptr(out_r), _ptr(out_c), _ptr(out_v), st), "sgap_mm_sum_runs")
    row_ptr = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    _native.check(L.sgap_mm_row_ptr(_ptr(out_r), nruns, rows, _ptr(row_ptr), st), "sgap_mm_row_ptr")
    return DeviceCoo(rows, cols, row_ptr, out_c, out_v)
