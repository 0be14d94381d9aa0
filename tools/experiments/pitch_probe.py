"""Shifted-block walk (variant 8) with pitch-ordered traversal (experiment):
SGAP_PITCH / SGAP_SEG read by sgap_run at each launch; bitwise check against
the linear order, interleaved timings on config 4."""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(4, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
rp = a.row_ptr.cpu().numpy().astype(np.int64)
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
cd = Candidate("row:8,col:4,r:1", 256, 0, 8)
k = plan_for(cd, n, a.num_rows, a.num_cols, rp)
aux = prepare_aux(k, a)
settings = [(0, 4, 128), (0, 4, 64)]
for blk in (128, 256):
    for seg in (1, 2, 4, 8):
        settings.append((160, seg, blk))
settings += [(320, 2, 128), (160, 40, 128)]
ref = None
times = {s: [] for s in settings}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rnd in range(5):
    order = settings if rnd % 2 == 0 else settings[::-1]
    for (pitch, seg, blk) in order:
        os.environ["SGAP_PITCH"] = str(pitch)
        os.environ["SGAP_SEG"] = str(seg)
        spmm(k, a, b, c, aux=aux, hw_block=blk, hw_variant=8)
        torch.cuda.synchronize()
        if rnd == 0:
            if ref is None:
                ref = c.clone()
            print(pitch, seg, blk, "bitwise", bool(torch.equal(c, ref)), flush=True)
        best = float("inf")
        for _ in range(3):
            e0.record()
            spmm(k, a, b, c, aux=aux, hw_block=blk, hw_variant=8)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        times[(pitch, seg, blk)].append(best)
base = statistics.median(times[settings[0]])
for s, ts in sorted(times.items(), key=lambda kv: statistics.median(kv[1])):
    m = statistics.median(ts)
    print(f"n={n} pitch={s[0]:4d} seg={s[1]:3d} blk={s[2]:4d} {m:8.3f} ms {m / base:6.3f}x", flush=True)
