"""One launch each of the reference kernel and ours for one point on config 2
(for an ncu side-by-side)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from baseline import refgen  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, device_block_starts, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

point = sys.argv[1] if len(sys.argv) > 1 else "row:1/32,col:1,r:32"
dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(2, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
n = 128
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
rp = a.row_ptr.cpu().numpy().astype(np.int64)
rk = refgen.find(point, n, 256)
k = plan_for(Candidate(point, 256), n, a.num_rows, a.num_cols, rp)
starts = device_block_starts(a, k.chunk, k.grid_size) if rk.has_block_starts else None
aux = prepare_aux(k, a)
torch.cuda.synchronize()
refgen.run(rk, k.grid_size, a, b, c, starts)
spmm(k, a, b, c, aux=aux)
torch.cuda.synchronize()
