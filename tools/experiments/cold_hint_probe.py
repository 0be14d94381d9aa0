"""Probe: streaming cache operator (ld.global.cs: evict-first in L1/L2) on the
B-row gathers of COLD columns (outside the top-H columns by gather count),
normal loads for the hot set -- hw variant 9 of the register walk, columns
flagged in bit 31 of a plan-owned copy of col_idx.  Same build, same box:
variant 1 on the plain matrix vs variant 9 on the flagged one, for several H."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--point", default="nnz:512,col:4,r:1")
ap.add_argument("--hot", default="32768,65536,131072,262144,524288")
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
stream = torch.cuda.current_stream()


def timed(aa, variant):
    k = plan_for(Candidate(args.point, 256, 0, variant), n, aa.num_rows, aa.num_cols, rp)
    aux = prepare_aux(k, aa)
    spmm(k, aa, b, c, aux=aux, hw_variant=variant)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(args.reps):
        e0.record(stream)
        spmm(k, aa, b, c, aux=aux, hw_variant=variant)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


base = timed(a, 1)
ref = c.clone()
print(desc, f"variant 1: {base:.3f} ms", flush=True)
counts = torch.bincount(a.col_idx.long(), minlength=a.num_cols)
order = torch.argsort(counts, descending=True)
cum = torch.cumsum(counts[order].double(), 0) / a.nnz
for H in [int(x) for x in args.hot.split(",")]:
    hot = torch.zeros(a.num_cols, dtype=torch.bool, device=dev)
    hot[order[:H]] = True
    flag = (~hot[a.col_idx.long()]).to(torch.int32) << 31
    col2 = a.col_idx | flag
    a2 = DeviceCsr(a.num_rows, a.num_cols, a.row_ptr, col2, a.vals)
    t = timed(a2, 9)
    diff = float((c - ref).abs().max().item())
    print(f"H={H} ({H * n * 4 / 1e6:.0f} MB hot, {float(cum[H - 1]):.2f} of gathers): variant 9 "
          f"{t:.3f} ms ({t / base:.3f}x), max|diff| {diff:.1e}", flush=True)
    del col2, a2, flag, hot
    torch.cuda.empty_cache()
