"""One variant-10 call and the contiguous-panel equivalent (four N=64 calls
on contiguous panels of B and C) back to back on config 3 at N=256, for an
ncu launch list (per-launch durations of k_panelize and every pass)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, _first_p, plan_for  # noqa: E402

dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(3, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
del g
rp = a.row_ptr.cpu().numpy().astype(np.int64)
pt = "nnz:512,col:4,r:1"
n, p = 256, 64
b = bench.dense_b(a.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), device=dev)
k = plan_for(Candidate(pt, _first_p(pt, n)), n, a.num_rows, a.num_cols, rp)
aux = prepare_aux(k, a, l2_hints=False)
kp = plan_for(Candidate(pt, _first_p(pt, p)), p, a.num_rows, a.num_cols, rp)
auxp = prepare_aux(kp, a)
bs = [b[:, i:i + p].contiguous() for i in range(0, n, p)]
cs = [torch.empty((a.num_rows, p), device=dev) for _ in bs]
for _ in range(2):
    spmm(k, a, b, c, aux=aux, hw_variant=10)
    torch.cuda.synchronize()
    for bi, ci in zip(bs, cs):
        spmm(kp, a, bi, ci, aux=auxp, hw_variant=1)
    torch.cuda.synchronize()
print("done", desc)
