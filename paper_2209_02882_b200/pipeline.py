"""Host-buffer SpMM with copies overlapped against compute (the e2e path).

``HostSpmm`` takes A and B in pinned host memory and returns C in pinned
host memory.  A is cut into nnz-balanced row blocks (``partition``); B goes
up first, then block b's (col, val) upload overlaps block b-1's SpMM, and
block b's C download (device->host, the other PCIe direction) overlaps block
b+1's upload and compute.  Device buffers are double-buffered across calls,
so call i+1's uploads run while call i's C is still coming down: back-to-back
calls approach max(H2D bytes, D2H bytes) / PCIe bandwidth.  Three CUDA
streams (in / compute / out) ordered by events; every block is a complete
SpMM on a row slice (rows are independent), so the result equals the
single-shot call.  ``wait(stream)`` orders a stream after all issued calls.
The sparsity structure is fixed per ``HostSpmm`` (each block's plan is bound
to it); values and B change per call.
"""

from __future__ import annotations

import torch

from .device import DeviceCsr, prepare_aux, spmm
from .lowering import LoweredKernel
from .partition import plan_shards

__all__ = ["HostSpmm"]


class HostSpmm:
    """Pipelined C = A @ B from pinned host buffers.

    The sparsity structure is fixed at construction (``h_rp``, ``h_ci``,
    pinned host tensors): every block is planned once per device buffer set
    (``sgap_plan`` binds a plan to its structure buffers), and every call
    still uploads the structure with the values, so a step moves all of A and
    B up and C down.  Only values may change between calls (``h_v``, ``h_b``).
    ``plan_fn(rows, row_ptr_host) -> LoweredKernel`` builds the kernel for a
    row block (the schedule is the caller's choice, e.g. selector output).
    """

    def __init__(self, num_rows: int, num_cols: int, n: int, h_rp: torch.Tensor,
                 h_ci: torch.Tensor, plan_fn, *, blocks: int = 4, device=None,
                 dtype=torch.float32, hw_variant: int = 0):
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.m, self.k, self.n, self.dtype = num_rows, num_cols, n, dtype
        rp = h_rp.numpy()
        self.plan = plan_shards(rp, max(1, blocks))
        self.h_ci = h_ci
        self.nnz = int(rp[-1])
        if h_ci.numel() != self.nnz:
            raise ValueError("col_idx length differs from row_ptr[-1]")
        self.hw_variant = hw_variant
        self.kernels: list[LoweredKernel] = []
        # rebased per-block row_ptr slices, pinned once (the structure is fixed)
        self.h_rps = []
        for g in range(self.plan.k):
            lo, hi = self.plan.rows(g)
            sub = (rp[lo:hi + 1] - rp[lo]).astype("int32")
            self.h_rps.append(torch.from_numpy(sub).pin_memory())
            self.kernels.append(plan_fn(hi - lo, sub))
        # two device buffer sets, each with its own plans (a plan is bound to
        # the structure buffers it was built on)
        self.sets = [self._buffers() for _ in range(2)]
        for d in self.sets:
            d["aux"] = []
            for g in range(self.plan.k):
                lo, hi = self.plan.rows(g)
                d["rp"][g].copy_(self.h_rps[g])
                b0, b1 = int(self.plan.nnz_begin[g]), int(self.plan.nnz_end[g])
                d["ci"][g][: b1 - b0].copy_(h_ci[b0:b1])
                a = self._csr(d, g)
                d["aux"].append(prepare_aux(self.kernels[g], a) if hi > lo else None)
        torch.cuda.synchronize(self.dev)
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.calls = 0

    def _csr(self, d: dict, g: int) -> DeviceCsr:
        lo, hi = self.plan.rows(g)
        cnt = self.plan.nnz(g)
        return DeviceCsr(hi - lo, self.k, d["rp"][g], d["ci"][g][:cnt], d["v"][g][:cnt])

    def _buffers(self) -> dict:
        # one allocation per block keeps every block's A arrays 16-byte aligned
        # (vectorised / bulk-copy walks need it; nnz-balanced cuts land anywhere)
        d = {"rp": [], "ci": [], "v": [],
             "b": torch.empty((self.k, self.n), dtype=self.dtype, device=self.dev),
             "c": torch.empty((self.m, self.n), dtype=self.dtype, device=self.dev),
             "cmp_done": None, "out_done": None}
        for g in range(self.plan.k):
            lo, hi = self.plan.rows(g)
            cnt = max(self.plan.nnz(g), 4)
            d["rp"].append(torch.empty(hi - lo + 1, dtype=torch.int32, device=self.dev))
            d["ci"].append(torch.empty(cnt, dtype=torch.int32, device=self.dev))
            d["v"].append(torch.empty(cnt, dtype=self.dtype, device=self.dev))
        return d

    def h2d_bytes(self) -> int:
        esz = torch.empty(0, dtype=self.dtype).element_size()
        rp_bytes = sum(t.numel() * 4 for t in self.h_rps)
        return rp_bytes + self.nnz * (4 + esz) + self.k * self.n * esz

    def d2h_bytes(self) -> int:
        return self.m * self.n * torch.empty(0, dtype=self.dtype).element_size()

    def wait(self, stream=None):
        """Order ``stream`` (default: current) after every issued call."""
        (stream or torch.cuda.current_stream(self.dev)).wait_stream(self.s_out)

    def __call__(self, h_v: torch.Tensor, h_b: torch.Tensor, h_c: torch.Tensor) -> torch.Tensor:
        """Values h_v (nnz), B h_b (K x n) and C h_c (M x n), all pinned; the
        structure given at construction is uploaded with them.  Stream-ordered
        after the caller's current stream; returns h_c (valid after
        synchronize)."""
        if h_v.numel() != self.nnz or tuple(h_b.shape) != (self.k, self.n) or \
                tuple(h_c.shape) != (self.m, self.n):
            raise ValueError("HostSpmm: values / B / C do not match the planned shapes")
        cur = torch.cuda.current_stream(self.dev)
        d = self.sets[self.calls % 2]
        self.calls += 1
        self.s_in.wait_stream(cur)
        if d["cmp_done"] is not None:  # inputs of this set free again (call i-2 computed)
            self.s_in.wait_event(d["cmp_done"])
        with torch.cuda.stream(self.s_in):
            d["b"].copy_(h_b, non_blocking=True)
        ev_in = []
        for g in range(self.plan.k):
            b0, b1 = int(self.plan.nnz_begin[g]), int(self.plan.nnz_end[g])
            with torch.cuda.stream(self.s_in):
                d["rp"][g].copy_(self.h_rps[g], non_blocking=True)
                if b1 > b0:
                    d["ci"][g][: b1 - b0].copy_(self.h_ci[b0:b1], non_blocking=True)
                    d["v"][g][: b1 - b0].copy_(h_v[b0:b1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(self.s_in)
                ev_in.append(e)
        if d["out_done"] is not None:  # C of this set downloaded (call i-2)
            self.s_cmp.wait_event(d["out_done"])
        ev_c = []
        for g in range(self.plan.k):
            lo, hi = self.plan.rows(g)
            self.s_cmp.wait_event(ev_in[g])
            with torch.cuda.stream(self.s_cmp):
                if hi > lo:
                    spmm(self.kernels[g], self._csr(d, g), d["b"], d["c"][lo:hi],
                         aux=d["aux"][g], hw_variant=self.hw_variant, stream=self.s_cmp)
                e = torch.cuda.Event()
                e.record(self.s_cmp)
                ev_c.append(e)
        d["cmp_done"] = ev_c[-1]
        for g in range(self.plan.k):
            lo, hi = self.plan.rows(g)
            self.s_out.wait_event(ev_c[g])
            with torch.cuda.stream(self.s_out):
                if hi > lo:
                    h_c[lo:hi].copy_(d["c"][lo:hi], non_blocking=True)
        out_done = torch.cuda.Event()
        out_done.record(self.s_out)
        d["out_done"] = out_done
        return h_c
