"""The executor: ``run`` executes a lowered kernel on the B200.

Drop-in for ``spmmlab.sim`` (``/root/reference/pkg/src/spmmlab/sim.py``):

  run(kernel, a, b, c0=None, *, precision="double") -> (DenseMatrix, metrics)
                                                      sim.py:431-487
  exec_seg_reduce_group / exec_atomic_add_group       sim.py:139-165 / 112-136
  SimulationFault                                     sim.py:63-70

The reference interprets LLIR on a 32-lane numpy model; here the same kernel
(identified by ``family`` + ``point``) runs as a hand-written sm_100a kernel in
``libsgap.so``.  Inputs are immutable, ``c0`` seeds C (C += A @ B) and is
copied, the result is a fresh float64 ``DenseMatrix``.  ``precision="single"``
computes in float32 (the production dtype), ``"double"`` in float64.
``kernel`` may be this package's ``LoweredKernel`` or the reference's (duck
typed on family/point/grid_size/block_size).

Metrics: ``atomic_ops`` is counted on the device and equals the reference
simulator's counter for the same kernel and matrix (a bit-exact pin, see
tests/test_gpu_parity.py); warp-step counters have no GPU meaning and are
replaced by the measured ``device_ms``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device import (DeviceCsr, host_cast, host_widen, native_dtype, prepare_aux, require_cuda,
                     spmm, torch_dtype, validate_csr)
from .lowering import LoweredKernel
from .matrices import DenseMatrix
from .space import parse_point
from .templates import algorithm_template
from .lowering import KernelConfig, lower

__all__ = ["WARP_LANES", "GpuMetrics", "SimulationFault", "exec_atomic_add_group",
           "exec_seg_reduce_group", "run", "resolve_kernel"]

WARP_LANES = 32


class SimulationFault(RuntimeError):
    """A group invariant was violated on the device (diverging indices in a
    parallel group, decreasing indices in a segment group, or an index out of
    range).  ``lane`` is the first offending lane."""

    def __init__(self, message: str, *, lane: int | None = None, node=None):
        super().__init__(message)
        self.lane = lane
        self.node = node


@dataclass(frozen=True)
class GpuMetrics:
    atomic_ops: int
    device_ms: float
    grid_size: int
    block_size: int
    family: str
    max_warp_steps: int | None = None
    total_steps: int | None = None
    idle_lane_steps: int | None = None

    def to_json(self) -> str:
        return json.dumps({
            "atomic_ops": self.atomic_ops, "device_ms": self.device_ms,
            "grid_size": self.grid_size, "block_size": self.block_size, "family": self.family,
            "max_warp_steps": None, "total_steps": None, "idle_lane_steps": None,
        })


def resolve_kernel(kernel, n: int, matrix) -> LoweredKernel:
    """Our LoweredKernel, rebuilt from a reference LoweredKernel if needed.

    The reference kernel carries family, point text, grid and block size; p
    is recovered from block_size (equal to p for three families, p*c^2/n for
    nnz-multiple)."""
    if isinstance(kernel, LoweredKernel):
        return kernel
    point = parse_point(kernel.point)
    c = point.col_amount.factor
    p = kernel.block_size
    if kernel.family == "nnz-multiple":
        p = kernel.block_size * n // (c * c)
    tpl = algorithm_template(point, KernelConfig(n=n, p=p))
    if tpl is None or tpl.family != kernel.family:
        raise ValueError(f"cannot map kernel {kernel.name} ({kernel.point}) onto a B200 template")
    ours = lower(tpl, matrix, name=kernel.name, compute_starts=False)
    if ours.grid_size != kernel.grid_size or ours.block_size != kernel.block_size:
        raise ValueError("kernel geometry does not match the matrix")
    return ours


def run(kernel, a, b, c0=None, *, precision: str = "double", device=None,
        hw_block: int = 0, hw_variant: int = 0) -> tuple[DenseMatrix, GpuMetrics]:
    """Execute ``kernel`` for C = c0 + A @ B on the GPU."""
    dt = torch_dtype(precision)  # ValueError on unknown precision, as in sim.py:444-445
    if a.num_cols != b.num_rows:
        raise ValueError(f"shape mismatch: A is {a.num_rows}x{a.num_cols}, B has {b.num_rows} rows")
    if kernel.block_size % WARP_LANES != 0:
        raise ValueError(f"block size {kernel.block_size} is not a warp multiple")
    n = int(b.num_cols)
    if c0 is not None and (c0.num_rows, c0.num_cols) != (a.num_rows, n):
        raise ValueError("output seed shape mismatch")
    k = resolve_kernel(kernel, n, a)
    if k.n != n:
        raise ValueError(f"kernel was lowered for n={k.n}, B has {n} columns")
    dev = require_cuda(device)
    np_dt = np.float32 if dt == torch.float32 else np.float64
    da = DeviceCsr.from_host(a, dtype=dt, device=dev)
    db = host_cast(b.vals, np_dt).reshape(a.num_cols, n).to(dev)
    if c0 is None:
        dc = torch.empty((a.num_rows, n), dtype=dt, device=dev)
    else:
        dc = host_cast(c0.vals, np_dt).reshape(a.num_rows, n).to(dev)  # a copy: c0 is not aliased
    wb = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    # the simulator faults on an out-of-range index (sim.py:279-287) instead of
    # reading out of bounds: the planner validates the CSR on the device first
    fault = validate_csr(da, stream=stream)
    if fault is not None:
        where = f"row_ptr[{-fault - 1}]" if fault < 0 else f"position {fault}"
        raise SimulationFault(f"malformed CSR operand at {where} (index out of range or "
                              "invariant broken)", lane=fault)
    aux = prepare_aux(k, da, stream=stream)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    spmm(k, da, db, dc, accumulate=c0 is not None, aux=aux, writebacks=wb,
         hw_block=hw_block, hw_variant=hw_variant, stream=stream)
    t1.record(stream)
    t1.synchronize()
    out = DenseMatrix(a.num_rows, n, host_widen(dc).reshape(-1))
    metrics = GpuMetrics(atomic_ops=int(wb.item()), device_ms=float(t0.elapsed_time(t1)),
                         grid_size=k.grid_size, block_size=k.block_size, family=k.family)
    return out, metrics


# --- group macros on the device (sim.py:112-165) -------------------------------


def _group_call(fn_name: str, idx, val, out, active, group_size: int) -> int:
    idx = np.asarray(idx, dtype=np.int64)
    val = np.asarray(val)
    if group_size < 1:
        raise ValueError("group size must be positive")
    if idx.shape[0] % group_size != 0:
        raise ValueError(f"lane count {idx.shape[0]} is not a multiple of group size {group_size}")
    if group_size > 32 or group_size & (group_size - 1):
        raise ValueError("the device group macros take group sizes 1, 2, 4, 8, 16 or 32")
    dev = require_cuda()
    out_arr = np.asarray(out)
    dt = torch.float32 if out_arr.dtype == np.float32 else torch.float64
    d_idx = torch.from_numpy(np.ascontiguousarray(idx)).to(dev)
    d_val = torch.from_numpy(np.ascontiguousarray(val, dtype=np.float32 if dt == torch.float32 else np.float64)).to(dev)
    d_act = None
    if active is not None:
        d_act = torch.from_numpy(np.ascontiguousarray(np.asarray(active, dtype=bool).astype(np.uint8))).to(dev)
    d_out = torch.from_numpy(np.ascontiguousarray(out_arr, dtype=np.float32 if dt == torch.float32 else np.float64)).to(dev)
    wb = torch.zeros(1, dtype=torch.int64, device=dev)
    fault = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
    import ctypes
    st = getattr(_native.lib(), fn_name)(
        d_idx.data_ptr(), d_val.data_ptr(), d_act.data_ptr() if d_act is not None else None,
        idx.shape[0], group_size, d_out.data_ptr(), out_arr.shape[0], native_dtype(dt),
        wb.data_ptr(), fault.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    _native.check(st, fn_name)
    lane = int(fault.item())
    if lane != np.iinfo(np.int64).max:
        g = lane // group_size
        kind = "segmented reduction with decreasing indices" if "seg" in fn_name else \
            "group atomic add with diverging indices"
        raise SimulationFault(f"{kind} in lane group {g}", lane=lane)
    out_arr[...] = d_out.cpu().numpy()
    return int(wb.item())


def exec_seg_reduce_group(idx, val, out, active=None, *, group_size: int) -> int:
    """Segmented group reduction on the device; returns the writeback count."""
    return _group_call("sgap_seg_reduce_group", idx, val, out, active, group_size)


def exec_atomic_add_group(idx, val, out, active=None, *, group_size: int) -> int:
    """Parallel group reduction on the device; returns the writeback count."""
    return _group_call("sgap_atomic_add_group", idx, val, out, active, group_size)
