"""Device-resident operands and the stream-ordered SpMM call.

PyTorch is used here only as plumbing -- device allocation, streams, events
and host<->device copies.  Every FLOP of the SpMM runs in ``libsgap.so``
(``include/sgap.h``), reached through ctypes with raw device pointers.

Device layout: ``row_ptr`` int32[M+1],
``col_idx`` int32[nnz], ``vals`` float32|float64[nnz]; B row-major [K, N];
C row-major [M, N]; all 64-bit element offsets inside the kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .lowering import LoweredKernel

__all__ = ["DeviceCsr", "KernelAux", "kernel_struct", "device_block_starts", "prepare_aux", "spmm",
           "launches_per_call", "reference_spmm_f64", "torch_dtype", "native_dtype", "require_cuda"]

_INT32_MAX = 2**31 - 1


def require_cuda(device=None) -> torch.device:
    """The product path runs on a CUDA device only -- fail loudly otherwise."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_02882_b200 needs a CUDA (sm_100a) device; none is visible")
    _native.lib()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    return dev


def torch_dtype(precision: str) -> torch.dtype:
    if precision == "single":
        return torch.float32
    if precision == "double":
        return torch.float64
    raise ValueError(f"unknown precision {precision!r}")


def native_dtype(t: torch.dtype) -> int:
    if t == torch.float32:
        return _native.F32
    if t == torch.float64:
        return _native.F64
    raise ValueError(f"unsupported value dtype {t}")


@dataclass
class DeviceCsr:
    """CSR operand resident in HBM (int32 indices)."""

    num_rows: int
    num_cols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    vals: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @property
    def device(self) -> torch.device:
        return self.row_ptr.device

    @classmethod
    def from_host(cls, a, *, dtype=torch.float32, device=None, non_blocking=False) -> "DeviceCsr":
        """Upload any CSR with num_rows/num_cols/row_ptr/col_idx/vals (ours
        or the reference's CsrMatrix)."""
        dev = require_cuda(device)
        rp = np.asarray(a.row_ptr)
        if rp[-1] > _INT32_MAX or a.num_rows >= _INT32_MAX:
            raise ValueError("nnz and num_rows must fit int32 on the device")
        ci = np.asarray(a.col_idx)
        vals = np.asarray(a.vals)
        np_dt = np.float32 if dtype == torch.float32 else np.float64

        def up(x, dt):
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=dt))
            if non_blocking:
                t = t.pin_memory()
            return t.to(dev, non_blocking=non_blocking)

        return cls(int(a.num_rows), int(a.num_cols), up(rp, np.int32), up(ci, np.int32),
                   up(vals, np_dt))

    def check(self) -> None:
        for name in ("row_ptr", "col_idx", "vals"):
            t = getattr(self, name)
            if not t.is_cuda:
                raise ValueError(f"DeviceCsr.{name} must be a CUDA tensor (got {t.device})")
            if not t.is_contiguous():
                raise ValueError(f"DeviceCsr.{name} must be contiguous")
        if self.row_ptr.dtype != torch.int32 or self.col_idx.dtype != torch.int32:
            raise ValueError("row_ptr and col_idx must be int32 on the device")
        if self.row_ptr.numel() != self.num_rows + 1:
            raise ValueError("row_ptr must have num_rows + 1 entries")

    def view(self) -> _native.Csr:
        self.check()
        return _native.Csr(self.num_rows, self.num_cols, self.nnz, self.row_ptr.data_ptr(),
                           self.col_idx.data_ptr(), self.vals.data_ptr())

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.row_ptr, self.col_idx, self.vals))

    def slice_rows(self, lo: int, hi: int) -> "DeviceCsr":
        """Rows [lo, hi) as a rebased CSR (device copy of the row_ptr slice;
        col/val are views).  Used by the row-shard partitioner."""
        rp = self.row_ptr[lo:hi + 1]
        base = int(rp[0].item())
        end = int(rp[-1].item())
        return DeviceCsr(hi - lo, self.num_cols, (rp - base).contiguous(), self.col_idx[base:end],
                         self.vals[base:end])


def kernel_struct(k: LoweredKernel, *, hw_block: int = 0, hw_variant: int = 0) -> _native.Kernel:
    fam = _native.FAMILY_IDS[k.family]
    return _native.Kernel(fam, k.n, k.p, k.g, k.c, k.r, k.chunk, k.grid_size, k.block_size,
                          1 if k.family in ("nnz-one", "nnz-multiple") else 0, hw_block, hw_variant)


def _stream_handle(stream) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def device_block_starts(a: DeviceCsr, chunk: int, num_blocks: int, *, stream=None) -> torch.Tensor:
    """lowering.compute_block_starts on the device (int32[num_blocks + 1])."""
    out = torch.empty(num_blocks + 1, dtype=torch.int32, device=a.device)
    _native.check(_native.lib().sgap_block_starts(a.row_ptr.data_ptr(), a.num_rows, chunk,
                                                  num_blocks, out.data_ptr(), _stream_handle(stream)),
                  "sgap_block_starts")
    return out


@dataclass
class KernelAux:
    """Per-(kernel, matrix) device side data: the block-start table
    (LoweredKernel.block_starts) and the float64 long-row table.  Built once
    by ``prepare_aux`` and reused across calls on the same matrix."""

    starts: torch.Tensor | None
    rowid: torch.Tensor | None = None
    long_rows: torch.Tensor | None = None
    long_count: torch.Tensor | None = None
    long_acc: torch.Tensor | None = None
    long_capacity: int = 0
    long_threshold: int = -1
    has_exact_rows: int = 0
    long_slot: torch.Tensor | None = None
    long_chunk: int = 0
    exact_rows: torch.Tensor | None = None

    def view(self) -> _native.Aux:
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        n_exact = int(self.exact_rows.numel()) if self.exact_rows is not None else 0
        return _native.Aux(ptr(self.starts), ptr(self.rowid), ptr(self.long_rows),
                           ptr(self.long_count), ptr(self.long_acc), self.long_capacity,
                           self.long_threshold, self.has_exact_rows, ptr(self.long_slot),
                           self.long_chunk, ptr(self.exact_rows), n_exact)

    def nbytes(self) -> int:
        ts = (self.starts, self.rowid, self.long_rows, self.long_count, self.long_acc,
              self.long_slot, self.exact_rows)
        return sum(t.numel() * t.element_size() for t in ts if t is not None)


def prepare_aux(k: LoweredKernel, a: DeviceCsr, *, stream=None, long_rows: bool = True,
                long_threshold: int | None = None, block_starts: bool = True,
                split_rows: bool = False, row_ptr_host=None) -> KernelAux:
    """Per-matrix side data of kernel ``k``: block starts and per-position row
    ids (nnz families) and, for float32 values, the long-row table
    (include/sgap.h: sgap_block_starts, sgap_row_ids, sgap_prepare_long_rows).

    ``split_rows``: nnz-multiple rows that straddle a g-chunk boundary also
    go to the float64 table (every split row summed in float64, no zero-fill
    pre-pass).  Off by default: on config 2 its float64 flushes cost more
    than the pre-pass they replace (0.764 vs 0.754 ms at g=512).

    ``row_ptr_host``: the same row_ptr on the host (numpy); given, planning
    never synchronises with the device (the longest-row check runs on it)."""
    eb = k.family in ("nnz-one", "nnz-multiple")
    a.check()
    starts = None
    if eb and k.grid_size > 0 and block_starts:
        starts = device_block_starts(a, k.chunk, k.grid_size, stream=stream)
    aux = KernelAux(starts)
    if not eb:
        return aux
    L = _native.lib()
    dev = a.device
    thr = -1
    chunk = 0
    if long_rows:
        ks = kernel_struct(k)
        thr = int(L.sgap_long_row_threshold(ctypes.byref(ks), native_dtype(a.vals.dtype)))
        if long_threshold is not None and thr >= 0:
            thr = int(long_threshold)
        if thr >= 0 and split_rows:
            chunk = int(L.sgap_long_row_chunk(ctypes.byref(ks), native_dtype(a.vals.dtype)))
    longest = 0
    lens = None
    if thr >= 0 and a.num_rows:  # does any row need the table?
        if row_ptr_host is not None:
            rph = np.asarray(row_ptr_host, dtype=np.int64)
        else:  # plan-time copy of row_ptr
            rph = a.row_ptr.cpu().numpy().astype(np.int64)
        lens = rph[1:] - rph[:-1]
        longest = int(lens.max())
        if longest <= thr and chunk == 0:
            thr = -1  # no long rows: no table, no fold launch
    aux.rowid = torch.empty(max(a.nnz, 4), dtype=torch.int32, device=dev)
    _native.check(L.sgap_row_ids(a.row_ptr.data_ptr(), a.num_rows, a.nnz, thr, chunk,
                                 aux.rowid.data_ptr(), _stream_handle(stream)), "sgap_row_ids")
    if thr < 0:
        return aux
    cap = int(L.sgap_long_row_capacity(a.nnz, thr, chunk))
    # rows k_row_ids flags exact (longer than the table threshold and the
    # error-free length), compacted for the error-free pass's grid
    if lens is not None and k.family == "nnz-multiple":
        exact = np.flatnonzero(lens > max(thr, int(L.sgap_exact_row_length()))).astype(np.int32)
        if exact.size:
            aux.exact_rows = torch.as_tensor(exact, device=dev)
    aux.has_exact_rows = int(aux.exact_rows is not None)
    aux.long_threshold = thr
    aux.long_chunk = chunk
    aux.long_capacity = cap
    aux.long_slot = torch.empty(max(a.num_rows, 1), dtype=torch.int32, device=dev)
    aux.long_rows = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    aux.long_count = torch.zeros(1, dtype=torch.int32, device=dev)
    aux.long_acc = torch.empty(max(cap, 1) * k.n, dtype=torch.float64, device=dev)
    tmp_bytes = int(L.sgap_long_rows_tmp_bytes(a.num_rows))
    tmp = torch.empty(max(tmp_bytes, 1), dtype=torch.uint8, device=dev)
    v = aux.view()
    _native.check(L.sgap_prepare_long_rows(a.row_ptr.data_ptr(), a.num_rows, k.n, ctypes.byref(v),
                                           tmp.data_ptr(), tmp_bytes, _stream_handle(stream)),
                  "sgap_prepare_long_rows")
    return aux


def spmm(k: LoweredKernel, a: DeviceCsr, b: torch.Tensor, c: torch.Tensor, *,
         accumulate: bool = False, aux: KernelAux | None = None,
         writebacks: torch.Tensor | None = None, hw_block: int = 0, hw_variant: int = 0,
         stream=None) -> None:
    """C (+)= A @ B with kernel ``k``, stream-ordered, no host synchronisation.

    ``b``: [num_cols, n] and ``c``: [num_rows, n] contiguous tensors of the
    value dtype of ``a``; ``aux`` from ``prepare_aux`` (built here when
    omitted -- pass it in to keep the call launch-only); ``writebacks``:
    optional int64[1] counter.
    """
    if b.dtype != a.vals.dtype or c.dtype != a.vals.dtype:
        raise ValueError("A, B and C must share one value dtype")
    if not (b.is_cuda and c.is_cuda):
        raise ValueError("B and C must be CUDA tensors")
    if tuple(b.shape) != (a.num_cols, k.n) or tuple(c.shape) != (a.num_rows, k.n):
        raise ValueError(
            f"shape mismatch: A is {a.num_rows}x{a.num_cols}, B {tuple(b.shape)}, C {tuple(c.shape)}, n={k.n}")
    if not (b.is_contiguous() and c.is_contiguous()):
        raise ValueError("B and C must be contiguous row-major")
    if aux is None:
        aux = prepare_aux(k, a, stream=stream)
    ks = kernel_struct(k, hw_block=hw_block, hw_variant=hw_variant)
    view = a.view()
    av = aux.view()
    st = _native.lib().sgap_run(
        ctypes.byref(ks), ctypes.byref(view), b.data_ptr(), c.data_ptr(),
        native_dtype(a.vals.dtype), 1 if accumulate else 0, ctypes.byref(av),
        writebacks.data_ptr() if writebacks is not None else None, _stream_handle(stream))
    _native.check(st, "sgap_run")


def launches_per_call(k: LoweredKernel, aux: KernelAux | None, *, accumulate: bool = False,
                      hw_variant: int = 0) -> int:
    """Kernels of libsgap.so one ``spmm`` call launches (the driver's memset
    for the nnz-one zero-fill is not ours and not counted)."""
    n = 1
    routed = aux is not None and aux.long_threshold >= 0 and aux.long_chunk == k.g
    if k.family == "nnz-multiple" and not accumulate and not routed:
        n += 1  # k_zero_shared_rows
    if aux is not None and aux.long_threshold >= 0 and k.family in ("nnz-one", "nnz-multiple"):
        n += 1  # k_long_rows_fold
        if k.family == "nnz-multiple" and aux.has_exact_rows:
            # the register walk takes exact chunks inline; the others launch
            # k_nnz_multiple_exact (sgap_api.cu run_nnz_multiple_w)
            w = min(32, max(1, k.n // k.c))
            variant = hw_variant or (2 if (w >= 16 and k.g <= 128) else 1)
            n += 0 if variant == 1 else 1
    return n


def reference_spmm_f64(a: DeviceCsr, b: torch.Tensor, n: int, *, stream=None) -> torch.Tensor:
    """The verify_point reference product in float64 on the device."""
    out = torch.empty((a.num_rows, n), dtype=torch.float64, device=a.device)
    view = a.view()
    st = _native.lib().sgap_reference_spmm_f64(ctypes.byref(view), b.data_ptr(), n,
                                               native_dtype(a.vals.dtype), out.data_ptr(),
                                               _stream_handle(stream))
    _native.check(st, "sgap_reference_spmm_f64")
    return out
