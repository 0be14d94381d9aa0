"""Time + error of one nnz-multiple point under different float64-table
thresholds (prepare_aux(long_threshold=...)) on a BASELINE config."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
import oracle  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--point", default="nnz:512,col:4,r:1")
ap.add_argument("--thresholds", default="0,2048,4096,8192,16384")
ap.add_argument("--variant", type=int, default=1)
args = ap.parse_args()
dev = torch.device("cuda", 0)
n = args.n or bench.default_n(args.config)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
rp = a.row_ptr.cpu().numpy().astype(np.int64)
want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(), a.vals.cpu().numpy(),
                       b.cpu().numpy(), n)
L = np.diff(rp)
k = plan_for(Candidate(args.point, 256), n, a.num_rows, a.num_cols, rp)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
print(desc, args.point)
for thr in [int(t) for t in args.thresholds.split(",")]:
    aux = prepare_aux(k, a, long_threshold=thr if thr > 0 else None)
    spmm(k, a, b, c, aux=aux, hw_variant=args.variant)
    best = 1e9
    for _ in range(5):
        e0.record(); spmm(k, a, b, c, aux=aux, hw_variant=args.variant); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    err = oracle.max_rel_error(c.cpu().numpy(), want)
    print(f"threshold {aux.long_threshold:6d} ({int((L > aux.long_threshold).sum())} rows, "
          f"{L[L > aux.long_threshold].sum() / L.sum():.2f} of nnz): {best:.3f} ms  err {err:.2e}")
