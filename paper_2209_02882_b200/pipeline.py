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
"""

from __future__ import annotations

import torch

from .device import DeviceCsr, prepare_aux, spmm
from .lowering import LoweredKernel
from .partition import plan_shards

__all__ = ["HostSpmm"]


class HostSpmm:
    """Pipelined C = A @ B from pinned host buffers.

    ``plan_fn(rows, row_ptr_host) -> LoweredKernel`` builds the kernel for a
    row block (the schedule is the caller's choice, e.g. selector output).
    """

    def __init__(self, num_rows: int, num_cols: int, n: int, row_ptr_host: torch.Tensor,
                 plan_fn, *, blocks: int = 4, device=None, dtype=torch.float32,
                 hw_variant: int = 0):
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.m, self.k, self.n, self.dtype = num_rows, num_cols, n, dtype
        rp = row_ptr_host.numpy() if isinstance(row_ptr_host, torch.Tensor) else row_ptr_host
        self.plan = plan_shards(rp, max(1, blocks))
        self.rp_host = row_ptr_host
        self.nnz = int(rp[-1])
        self.hw_variant = hw_variant
        self.kernels: list[LoweredKernel] = []
        for g in range(self.plan.k):
            lo, hi = self.plan.rows(g)
            sub = rp[lo:hi + 1] - rp[lo]
            self.kernels.append(plan_fn(hi - lo, sub))
        # device buffers (reused across calls)
        self.sets = [self._buffers() for _ in range(2)]
        # per-block side data (row ids, long-row table, block starts) depends
        # on the structure only: planned once here from a one-time copy of
        # each block's row_ptr, like runner.build_kernel's block_starts, and
        # reused by every call (the calls still upload all of A and B)
        self.auxes = []
        for g in range(self.plan.k):
            lo, hi = self.plan.rows(g)
            sub = (rp[lo:hi + 1] - rp[lo]).astype("int32")
            d0 = self.sets[0]
            a = DeviceCsr(hi - lo, self.k, torch.from_numpy(sub).to(self.dev),
                          d0["ci"][g][: self.plan.nnz(g)], d0["v"][g][: self.plan.nnz(g)])
            self.auxes.append(prepare_aux(self.kernels[g], a, row_ptr_host=sub) if hi > lo else None)
        torch.cuda.synchronize(self.dev)
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.calls = 0

    def _buffers(self) -> dict:
        # one allocation per block keeps every block's A arrays 16-byte aligned
        # (vectorised / bulk-copy walks need it; nnz-balanced cuts land anywhere)
        d = {"rp": torch.empty(self.m + 1, dtype=torch.int32, device=self.dev),
             "ci": [], "v": [],
             "b": torch.empty((self.k, self.n), dtype=self.dtype, device=self.dev),
             "c": torch.empty((self.m, self.n), dtype=self.dtype, device=self.dev),
             "cmp_done": None, "out_done": None}
        for g in range(self.plan.k):
            cnt = max(self.plan.nnz(g), 4)
            d["ci"].append(torch.empty(cnt, dtype=torch.int32, device=self.dev))
            d["v"].append(torch.empty(cnt, dtype=self.dtype, device=self.dev))
        return d

    def h2d_bytes(self) -> int:
        esz = torch.empty(0, dtype=self.dtype).element_size()
        return (self.m + 1) * 4 + self.nnz * (4 + esz) + self.k * self.n * esz

    def d2h_bytes(self) -> int:
        return self.m * self.n * torch.empty(0, dtype=self.dtype).element_size()

    def wait(self, stream=None):
        """Order ``stream`` (default: current) after every issued call."""
        (stream or torch.cuda.current_stream(self.dev)).wait_stream(self.s_out)

    def __call__(self, h_rp: torch.Tensor, h_ci: torch.Tensor, h_v: torch.Tensor, h_b: torch.Tensor,
                 h_c: torch.Tensor) -> torch.Tensor:
        """All host tensors pinned; h_c receives C.  Stream-ordered after the
        caller's current stream; returns h_c (valid after synchronize)."""
        cur = torch.cuda.current_stream(self.dev)
        d = self.sets[self.calls % 2]
        self.calls += 1
        self.s_in.wait_stream(cur)
        if d["cmp_done"] is not None:  # inputs of this set free again (call i-2 computed)
            self.s_in.wait_event(d["cmp_done"])
        with torch.cuda.stream(self.s_in):
            d["rp"].copy_(h_rp, non_blocking=True)
            d["b"].copy_(h_b, non_blocking=True)
        ev_in = []
        for g in range(self.plan.k):
            b0, b1 = int(self.plan.nnz_begin[g]), int(self.plan.nnz_end[g])
            with torch.cuda.stream(self.s_in):
                if b1 > b0:
                    d["ci"][g][: b1 - b0].copy_(h_ci[b0:b1], non_blocking=True)
                    d["v"][g][: b1 - b0].copy_(h_v[b0:b1], non_blocking=True)
                e = torch.cuda.Event()
                e.record(self.s_in)
                ev_in.append(e)
        if d["out_done"] is not None:  # C of this set downloaded (call i-2)
            self.s_cmp.wait_event(d["out_done"])
        ev_c = []
        for g in range(self.plan.k):
            lo, hi = self.plan.rows(g)
            b0, b1 = int(self.plan.nnz_begin[g]), int(self.plan.nnz_end[g])
            self.s_cmp.wait_event(ev_in[g])
            with torch.cuda.stream(self.s_cmp):
                rp = (d["rp"][lo:hi + 1] - b0).contiguous()
                a = DeviceCsr(hi - lo, self.k, rp, d["ci"][g][: b1 - b0], d["v"][g][: b1 - b0])
                k = self.kernels[g]
                if hi > lo:
                    spmm(k, a, d["b"], d["c"][lo:hi], aux=self.auxes[g],
                         hw_variant=self.hw_variant, stream=self.s_cmp)
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
