"""Probe: does an L2 set-aside (persisting window) over a compact copy of the
hottest B rows raise config 5's L2 hit rate where per-access evict_last hints
did not (profiles/r02_cfg5_memory_experiments.md, experiment 2)?

Bx = [B[hot] ; B]; col2 = hot ? slot : col + H, so the product kernel runs
unchanged on (col2, Bx); the first H rows of Bx sit in an access-policy window
(hitProp persisting) with cudaLimitPersistingL2CacheSize set.  Times the SpMM
for H in a list, with and without the window, on the same build and box.
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--point", default="nnz:512,col:4,r:1")
ap.add_argument("--hw-variant", type=int, default=1)
ap.add_argument("--hot", default="0,65536,131072,196608")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

dev = torch.device("cuda", 0)
n = bench.default_n(args.config)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
del g
torch.cuda.empty_cache()
b = bench.dense_b(a.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
rp = a.row_ptr.cpu().numpy().astype(np.int64)
k = plan_for(Candidate(args.point, 256, 0, args.hw_variant), n, a.num_rows, a.num_cols, rp)
counts = torch.bincount(a.col_idx.long(), minlength=a.num_cols)
order = torch.argsort(counts, descending=True)
cum = torch.cumsum(counts[order].double(), 0) / a.nnz
err, max_persist = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err, max_win = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
err, l2 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
print(desc, "L2", l2, "max persisting", max_persist, "max window", max_win, flush=True)
stream = torch.cuda.current_stream()


def time_it(aa, bb):
    kk = plan_for(Candidate(args.point, 256, 0, args.hw_variant), n, aa.num_rows, aa.num_cols, rp)
    aux = prepare_aux(kk, aa)
    spmm(kk, aa, bb, c, aux=aux, hw_variant=args.hw_variant)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(args.reps):
        e0.record(stream)
        spmm(kk, aa, bb, c, aux=aux, hw_variant=args.hw_variant)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def set_window(ptr, nbytes, ratio):
    v = rt.cudaStreamAttrValue()
    v.accessPolicyWindow.base_ptr = ptr
    v.accessPolicyWindow.num_bytes = nbytes
    v.accessPolicyWindow.hitRatio = ratio
    v.accessPolicyWindow.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    v.accessPolicyWindow.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    st = rt.cudaStreamSetAttribute(stream.cuda_stream,
                                   rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, v)
    return st


base = time_it(a, b)
ref = c.clone()
print(f"plain: {base:.3f} ms", flush=True)
for H in [int(x) for x in args.hot.split(",")]:
    if H == 0:
        continue
    hot = order[:H]
    share = float(cum[H - 1])
    slot = torch.full((a.num_cols,), -1, dtype=torch.int64, device=dev)
    slot[hot] = torch.arange(H, device=dev)
    ci = a.col_idx.long()
    s = slot[ci]
    col2 = torch.where(s >= 0, s, ci + H).to(torch.int32)
    bx = torch.cat([b[hot], b], 0)
    a2 = DeviceCsr(a.num_rows, a.num_cols + H, a.row_ptr, col2, a.vals)
    t_nowin = time_it(a2, bx)
    hot_bytes = H * n * 4
    for limit_frac in (0.5, 0.75, 1.0):
        lim = int(min(max_persist, hot_bytes) * limit_frac) if max_persist else 0
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, lim)
        win = min(hot_bytes, max_win)
        ratio = min(1.0, lim / win) if win else 0.0
        st = set_window(bx.data_ptr(), win, ratio)
        t_win = time_it(a2, bx)
        diff = float((c - ref).abs().max().item())
        set_window(0, 0, 0.0)
        rt.cudaCtxResetPersistingL2Cache()
        print(f"H={H} ({hot_bytes / 1e6:.0f} MB, {share:.2f} of gathers): remapped {t_nowin:.3f} ms, "
              f"window {win / 1e6:.0f} MB limit {lim / 1e6:.0f} MB ratio {ratio:.2f}: {t_win:.3f} ms "
              f"(set {st}, max|diff| {diff:.1e})", flush=True)
    del bx, col2, a2
    torch.cuda.empty_cache()
rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, 0)
