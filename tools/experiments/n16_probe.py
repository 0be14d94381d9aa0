"""Shifted sub-warp walk at N/c = 4 (N = 16): 8 lane groups of 4 rows (32-row
blocks) or of 2 rows (SGAP_SHIFT_R2, 16-row blocks) vs variant 4, config 4."""
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(4, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
rp = a.row_ptr.cpu().numpy().astype(np.int64)
n = 16
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
k = plan_for(Candidate("row:4,col:4,r:1", 256, 0, 4), n, a.num_rows, a.num_cols, rp)
aux = prepare_aux(k, a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
modes = [("v4", 4, False), ("v8 R4", 8, False), ("v8 R2", 8, True)]
times = {m[0]: [] for m in modes}
ref = None
for rnd in range(7):
    for name, v, r2 in (modes if rnd % 2 == 0 else modes[::-1]):
        if r2:
            os.environ["SGAP_SHIFT_R2"] = "1"
        else:
            os.environ.pop("SGAP_SHIFT_R2", None)
        spmm(k, a, b, c, aux=aux, hw_variant=v)
        torch.cuda.synchronize()
        if rnd == 0:
            if ref is None:
                ref = c.clone()
            print(name, "bitwise", bool(torch.equal(ref, c)))
        best = float("inf")
        for _ in range(3):
            e0.record()
            spmm(k, a, b, c, aux=aux, hw_variant=v)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        times[name].append(best)
for m, ts in times.items():
    print(m, f"{statistics.median(ts):.3f} ms")
