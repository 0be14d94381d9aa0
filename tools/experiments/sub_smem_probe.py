"""Shifted sub-warp walk at N/c = 16: values shuffled from registers vs read
from a shared slab (SGAP_SUB_SMEM, experiment), interleaved, config 4 N=64."""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
k = plan_for(Candidate("row:8,col:4,r:1", 256, 0, 8), n, a.num_rows, a.num_cols, rp)
aux = prepare_aux(k, a)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
times = {"shfl": [], "smem": []}
ref = None
for rnd in range(7):
    for mode in (("shfl", "smem") if rnd % 2 == 0 else ("smem", "shfl")):
        if mode == "smem":
            os.environ["SGAP_SUB_SMEM"] = "1"
        else:
            os.environ.pop("SGAP_SUB_SMEM", None)
        spmm(k, a, b, c, aux=aux, hw_variant=8)
        torch.cuda.synchronize()
        if ref is None:
            ref = c.clone()
        elif rnd == 0:
            print("bitwise", bool(torch.equal(ref, c)))
        best = float("inf")
        for _ in range(3):
            e0.record()
            spmm(k, a, b, c, aux=aux, hw_variant=8)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        times[mode].append(best)
for m, ts in times.items():
    print(m, f"{statistics.median(ts):.3f} ms")
