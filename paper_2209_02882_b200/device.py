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

__all__ = ["host_cast", "host_widen", "DeviceCsr", "KernelAux", "SpmmGraph", "kernel_struct", "device_block_starts", "prepare_aux", "spmm",
           "plan_workspace_bytes", "validate_csr", "spmm_rbpr_grid",
           "launches_per_call", "reference_spmm_f64", "torch_dtype", "native_dtype", "require_cuda"]

_INT32_MAX = 2**31 - 1


_TORCH_DT = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
             np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64}


def host_cast(x, dt) -> torch.Tensor:
    """A contiguous host tensor of numpy dtype ``dt`` from array-like ``x``;
    the element conversion runs on torch's CPU thread pool (the reference's
    float64 / int64 host layout to the device layout: config 5's 8.6 GB B
    takes ~2.8 s through numpy's single-threaded astype)."""
    a = np.asarray(x)
    if not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    t = torch.from_numpy(a)
    want = _TORCH_DT[np.dtype(dt)]
    return t if t.dtype == want else t.to(want)


def host_widen(t: torch.Tensor) -> np.ndarray:
    """Device result -> float64 numpy on the host: download in the value
    dtype (half the bytes for float32), widen on the CPU thread pool."""
    h = t.cpu()
    return (h if h.dtype == torch.float64 else h.to(torch.float64)).numpy()


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
            t = host_cast(x, dt)
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
    """The plan of one (kernel, matrix structure) pair: ``sgap_plan_t`` plus
    the device workspace it points into (block starts, per-position row ids,
    the float64 long-row table, the error-free row list), all built on the
    device by ``sgap_plan`` (include/sgap.h).  Reused across calls on the same
    structure; values, B and C may change between calls."""

    plan: _native.Plan
    workspace: torch.Tensor
    num_rows: int
    nnz: int

    @property
    def long_threshold(self) -> int:
        return int(self.plan.aux.long_threshold)

    @property
    def long_chunk(self) -> int:
        return int(self.plan.aux.long_chunk)

    @property
    def has_exact_rows(self) -> int:
        return int(self.plan.aux.has_exact_rows)

    @property
    def exact_count(self) -> int:
        return int(self.plan.aux.exact_count)

    @property
    def table_rows(self) -> int:
        return int(self.plan.table_rows)

    @property
    def longest_row(self) -> int:
        return int(self.plan.longest_row)

    @property
    def starts(self) -> torch.Tensor | None:
        """LoweredKernel.block_starts as computed on the device (int32)."""
        ptr = self.plan.aux.d_block_starts
        if not ptr:
            return None
        off = ptr - self.workspace.data_ptr()
        n = int(self.plan.kernel.grid_size) + 1
        return self.workspace[off:off + 4 * n].view(torch.int32)

    def nbytes(self) -> int:
        return int(self.workspace.numel())


# B larger than this (1.5x the 126 MB L2) gets cold-column hints by default
# (config 3 at N=256, B = 238 MB: variant 9 -3.2%, profiles/r02_ab_hints_cfg3_n256.log)
_L2_HINT_MIN_B_BYTES = 192 << 20
L2_DEVICE_BYTES = 132_644_864  # B200 cudaDevAttrL2CacheSize (what the planner reads)


def plan_workspace_bytes(k: LoweredKernel, a: DeviceCsr, *, split_rows: bool = False,
                         flags: int | None = None) -> int:
    ks = kernel_struct(k)
    view = a.view()
    out = ctypes.c_size_t(0)
    if flags is None:
        flags = _native.PLAN_SPLIT_ROWS if split_rows else 0
    _native.check(_native.lib().sgap_plan_workspace_bytes(
        ctypes.byref(ks), ctypes.byref(view), native_dtype(a.vals.dtype), flags,
        ctypes.byref(out)), "sgap_plan_workspace_bytes")
    return int(out.value)


def panel_lanes(num_cols: int, n: int, c: int, esz: int = 4, l2_bytes: int = L2_DEVICE_BYTES) -> int:
    """hw variant 10's panel width in c-wide column tiles, as the planner
    picks it (sgap_api.cu panel_lanes): the widest of 32 / 16 / 8 tiles
    (fewer than n / c) whose num_cols B rows fit half the L2; 0 when none
    does or the whole of B fits the L2."""
    if num_cols * n * esz <= l2_bytes:
        return 0
    for w in (32, 16, 8):
        if w < n // c and num_cols * w * c * esz <= l2_bytes // 2:
            return w
    return 0


def prepare_aux(k: LoweredKernel, a: DeviceCsr, *, stream=None, split_rows: bool = False,
                validate: bool = False, l2_hints: bool | None = None,
                panels: bool | None = None, row_ptr_host=None) -> KernelAux:
    """``sgap_plan``: the per-matrix half of ``runner.build_kernel``
    (block_starts, lowering.py:683-696) plus the engine's side data, built on
    the device in one workspace (one 24-byte read-back of row statistics).

    ``split_rows``: nnz-multiple rows that straddle a g-chunk boundary also
    go to the float64 table (no zero-fill pre-pass; measured slower on config
    2, off by default).  ``validate``: check the CsrMatrix invariants first
    (``sgap_validate_csr``; raises ``SimulationFault``-compatible
    ``SgapError`` status FAULT).  ``row_ptr_host`` is accepted for
    compatibility and unused: planning needs no host copy of the matrix.
    ``l2_hints``: build the cold-column cache hints of hw variant 9
    (nnz-multiple); None = when B is more than 1.5x the L2 (configs 3 at N=256, 5).
    ``panels``: reserve the panel-major copy of B that hw variant 10 walks
    (nnz-multiple; num_cols x n elements of workspace, only when B exceeds
    the L2 and a panel fits half of it); None = whenever that applies."""
    del row_ptr_host
    a.check()
    L = _native.lib()
    if l2_hints is None:
        l2_hints = (k.family == "nnz-multiple" and
                    a.num_cols * k.n * a.vals.element_size() > _L2_HINT_MIN_B_BYTES)
    if panels is None:
        panels = (k.family == "nnz-multiple" and
                  panel_lanes(a.num_cols, k.n, k.c, a.vals.element_size()) > 0)
    flags = ((_native.PLAN_SPLIT_ROWS if split_rows else 0) |
             (_native.PLAN_VALIDATE if validate else 0) |
             (_native.PLAN_L2_HINTS if l2_hints else 0) |
             (_native.PLAN_PANELS if panels else 0))
    ks = kernel_struct(k)
    view = a.view()
    nbytes = plan_workspace_bytes(k, a, flags=flags)
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=a.device)
    plan = _native.Plan()
    _native.check(L.sgap_plan(ctypes.byref(ks), ctypes.byref(view), native_dtype(a.vals.dtype),
                              flags, ws.data_ptr(), ws.numel(), ctypes.byref(plan),
                              _stream_handle(stream)), "sgap_plan")
    return KernelAux(plan, ws, a.num_rows, a.nnz)


def validate_csr(a: DeviceCsr, *, stream=None) -> int | None:
    """The CsrMatrix invariants on the device (matrices.py:58-75); None when
    valid, else the first offending position (a row_ptr index r as -(r+1))."""
    scratch = torch.empty(8, dtype=torch.uint8, device=a.device)
    pos = ctypes.c_int64(0)
    view = _native.Csr(a.num_rows, a.num_cols, a.nnz, a.row_ptr.data_ptr(), a.col_idx.data_ptr(),
                       a.vals.data_ptr())
    st = _native.lib().sgap_validate_csr(ctypes.byref(view), scratch.data_ptr(), ctypes.byref(pos),
                                         _stream_handle(stream))
    if st == _native.ERR_FAULT:
        return int(pos.value)
    _native.check(st, "sgap_validate_csr")
    return None


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
    ks = kernel_struct(k)
    pk = aux.plan.kernel
    if (pk.family, pk.n, pk.g, pk.c, pk.r, pk.chunk, pk.grid_size) != \
            (ks.family, ks.n, ks.g, ks.c, ks.r, ks.chunk, ks.grid_size):
        raise ValueError("the plan was built for another kernel")
    plan = _native.Plan.from_buffer_copy(aux.plan)
    plan.kernel.hw_block = hw_block
    plan.kernel.hw_variant = hw_variant
    view = a.view()
    st = _native.lib().sgap_run(
        ctypes.byref(plan), ctypes.byref(view), b.data_ptr(), c.data_ptr(),
        1 if accumulate else 0, writebacks.data_ptr() if writebacks is not None else None,
        _stream_handle(stream))
    _native.check(st, "sgap_run")


def spmm_rbpr_grid(k: LoweredKernel, a: DeviceCsr, b: torch.Tensor, c: torch.Tensor, *,
                   block: int, tile: int, worker_scale: float, accumulate: bool = False,
                   aux: KernelAux | None = None, writebacks: torch.Tensor | None = None,
                   stream=None) -> None:
    """The dgSPARSE RB+PR+RM kernel under one fine-grained tuning cell
    <groupSz = k.g, blockSz, tileSz, workerDimR = worker_scale x M>
    (space.FineGrainedConfig) for a row-reciprocal
    kernel ``k`` (row:1/g,col:c,r:g).  Same result as ``spmm(k, ...)``."""
    if k.family != "row-reciprocal":
        raise ValueError("the fine-grained RB+PR grid runs row-reciprocal kernels")
    if b.dtype != a.vals.dtype or c.dtype != a.vals.dtype:
        raise ValueError("A, B and C must share one value dtype")
    if tuple(b.shape) != (a.num_cols, k.n) or tuple(c.shape) != (a.num_rows, k.n):
        raise ValueError("shape mismatch")
    if not (b.is_contiguous() and c.is_contiguous()):
        raise ValueError("B and C must be contiguous row-major")
    if aux is None:
        aux = prepare_aux(k, a, stream=stream)
    view = a.view()
    st = _native.lib().sgap_run_rbpr_grid(
        ctypes.byref(aux.plan), ctypes.byref(view), b.data_ptr(), c.data_ptr(), block, tile,
        float(worker_scale), 1 if accumulate else 0,
        writebacks.data_ptr() if writebacks is not None else None, _stream_handle(stream))
    _native.check(st, "sgap_run_rbpr_grid")


class SpmmGraph:
    """One planned SpMM call captured as a CUDA graph and replayed: for
    repeated products on the same structure (iterative solvers, GNN layers)
    the whole call -- zero-fill, walk, long-row fold -- becomes one graph
    launch with no per-kernel host work.  ``sgap_run`` neither allocates nor
    synchronises, so it is capturable once the plan exists.  The captured
    call reads ``a.vals`` / ``b`` and writes ``c`` at their current
    addresses: update those tensors in place between replays."""

    def __init__(self, k: LoweredKernel, a: DeviceCsr, b: torch.Tensor, c: torch.Tensor, *,
                 aux: KernelAux | None = None, accumulate: bool = False, hw_block: int = 0,
                 hw_variant: int = 0):
        self.k, self.a, self.b, self.c = k, a, b, c
        self.aux = aux if aux is not None else prepare_aux(k, a)
        side = torch.cuda.Stream(a.device)
        side.wait_stream(torch.cuda.current_stream(a.device))
        with torch.cuda.stream(side):  # warm-up outside the capture (lazy loading)
            spmm(k, a, b, c, accumulate=accumulate, aux=self.aux, hw_block=hw_block,
                 hw_variant=hw_variant, stream=side)
        torch.cuda.current_stream(a.device).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            spmm(k, a, b, c, accumulate=accumulate, aux=self.aux, hw_block=hw_block,
                 hw_variant=hw_variant, stream=torch.cuda.current_stream(a.device))

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.c


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
            n += 0 if variant in (1, 5, 9, 10) else 1
    if k.family == "row-multiple" and hw_variant in (3, 4, 8) and k.c and k.n // k.c > 32:
        n += k.n // k.c // 32 - 1  # one warp-per-row pass per 32c-column panel
    if k.family == "nnz-multiple" and hw_variant == 10 and aux is not None:
        lanes = int(aux.plan.aux.panel_lanes)
        if lanes:  # k_panelize + one walk per column panel (the walk is counted above)
            n += 1 + (k.n + lanes * k.c - 1) // (lanes * k.c) - 1
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
