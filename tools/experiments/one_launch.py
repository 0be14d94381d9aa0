"""Plan + warm + one more launch of one schedule point on a BASELINE config
(the target of an `ncu --launch-skip 1 --launch-count 1` capture)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--point", default="nnz:512,col:4,r:1")
ap.add_argument("--p", type=int, default=256)
ap.add_argument("--variant", type=int, default=0)
args = ap.parse_args()
dev = torch.device("cuda", 0)
n = args.n or bench.default_n(args.config)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
k = plan_for(Candidate(args.point, args.p), n, a.num_rows, a.num_cols,
             a.row_ptr.cpu().numpy().astype(np.int64))
aux = prepare_aux(k, a)
for _ in range(2):
    spmm(k, a, b, c, aux=aux, hw_variant=args.variant)
torch.cuda.synchronize()
print(desc, args.point, "ok")
