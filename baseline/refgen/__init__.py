"""The reference compiler's emitted CUDA kernels on the B200.

``spmmlab.cuda.emit_cuda`` (cuda.py:91-183) turns a lowered schedule point
into CUDA text whose group macros are declared but not defined.  The texts
for every templated point at (n, p) in {(4,256), (32,256), (128,256)} are
frozen in tests/golden/refgen/ (tests/golden/make_refgen.py);
baseline/refgen/gen_tu.py wraps them with macro bodies that follow the
simulator (sim.py:112-165) and builds librefgen.so.  This is the
fixed-schedule "naive TACO" baseline: the reference's own kernels, same
schedule knobs, same launch geometry (grid/block from runner.build_kernel,
block starts from lowering.compute_block_starts), one (i, k) cell per lane,
no vectorisation.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
LIB_PATH = HERE / "librefgen.so"
MANIFEST = ROOT / "tests" / "golden" / "refgen" / "manifest.json"


@dataclass(frozen=True)
class RefKernel:
    point: str
    n: int
    p: int
    family: str
    kernel: str
    id: str
    block_size: int
    has_block_starts: bool
    da_spmm_corner: bool


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing -- run __graft_entry__.build()")
        L = ctypes.CDLL(str(LIB_PATH))
        vp = ctypes.c_void_p
        L.refgen_count.restype = ctypes.c_int
        L.refgen_launch.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_int,
                                    vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp]
        L.refgen_launch.restype = ctypes.c_int
        _lib = L
    return _lib


def kernels() -> list[RefKernel]:
    data = json.loads(MANIFEST.read_text())
    return [RefKernel(**e) for e in data["kernels"]]


def find(point: str, n: int, p: int) -> RefKernel | None:
    for k in kernels():
        if k.point == point and k.n == n and k.p == p:
            return k
    return None


def run(rk: RefKernel, grid_size: int, a, b: torch.Tensor, c: torch.Tensor,
        block_starts: torch.Tensor | None, *, zero: bool = True, stream=None) -> None:
    """C = A @ B with the reference's kernel ``rk`` (C zero-filled first, as
    sim.run seeds C with zeros; every emitted family accumulates into C).
    ``a``: paper_2209_02882_b200.device.DeviceCsr (int32 indices)."""
    if b.dtype != a.vals.dtype or c.dtype != a.vals.dtype:
        raise ValueError("A, B and C must share one value dtype")
    dtype = {torch.float32: 0, torch.float64: 1}[a.vals.dtype]
    if rk.has_block_starts and block_starts is None:
        raise ValueError(f"{rk.point}: block starts required")
    if tuple(b.shape) != (a.num_cols, rk.n) or tuple(c.shape) != (a.num_rows, rk.n):
        raise ValueError("shape mismatch")
    st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    if zero:
        c.zero_()
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    err = lib().refgen_launch(rk.id.encode(), dtype, grid_size, rk.block_size, ptr(a.row_ptr),
                              ptr(a.col_idx), ptr(a.vals), ptr(b), ptr(c), ptr(block_starts),
                              a.num_rows, rk.n, st)
    if err != 0:
        raise RuntimeError(f"refgen_launch({rk.point}, n={rk.n}, p={rk.p}) failed: {err}")
