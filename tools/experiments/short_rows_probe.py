"""Probe: on config 2 (R-MAT s20, N=128) with the rows longer than --cap
removed, is the warp-per-row RB walk (row-multiple variant 4, lane-staged A)
faster than the EB register walk (variants 5 / 1)?  If so, a hybrid (short
rows RB, long rows EB) could beat the EB walk on the full matrix.  Also
times both on the full matrix for reference."""
import argparse
import statistics
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
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--cap", type=int, default=64)
args = ap.parse_args()
dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
full = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
                 g.vals.to(torch.float32))
rp = g.row_ptr.long()
lens = rp[1:] - rp[:-1]
keep_row = lens <= args.cap
pos_row = torch.repeat_interleave(torch.arange(g.num_rows, device=dev), lens)
keep = keep_row[pos_row]
new_lens = torch.where(keep_row, lens, torch.zeros_like(lens))
new_rp = torch.zeros(g.num_rows + 1, dtype=torch.int64, device=dev)
new_rp[1:] = torch.cumsum(new_lens, 0)
short = DeviceCsr(g.num_rows, g.num_cols, new_rp.to(torch.int32), g.col_idx[keep].to(torch.int32),
                  g.vals[keep].to(torch.float32))
print(desc, "full nnz", full.nnz, "short-row nnz", short.nnz,
      f"({100 * short.nnz / full.nnz:.1f}%), rows > {args.cap}: {int((~keep_row).sum())}")
n = args.n
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((g.num_rows, n), device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, a in (("short rows", short), ("full", full)):
    rph = a.row_ptr.cpu().numpy().astype(np.int64)
    for text in ("nnz:512,col:4,r:1@256/5", "nnz:512,col:4,r:1@256/1", "row:1,col:4,r:1@256/4",
                 "row:4,col:4,r:1@256/4", "row:8,col:4,r:1@256/4"):
        pt, rest = text.split("@")
        p, v = rest.split("/")
        k = plan_for(Candidate(pt, int(p), 0, int(v)), n, a.num_rows, a.num_cols, rph)
        aux = prepare_aux(k, a)
        spmm(k, a, b, c, aux=aux, hw_variant=int(v))
        ts = []
        for _ in range(7):
            e0.record()
            spmm(k, a, b, c, aux=aux, hw_variant=int(v))
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{name:10s} {text:28s} {statistics.median(ts):.3f} ms", flush=True)
