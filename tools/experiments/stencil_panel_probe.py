"""Config 4 at wide N (256 / 512): one SpMM over all N columns against N/128
separate SpMMs over contiguous 128-column panels of B and C (the warp-per-row
walk at N/c = 32), which bounds what a column-panel mode of the RB walks could
gain (each panel pass keeps the stencil's sliding B window -- rows within one
z-plane of the current rows -- 4x smaller in L2).  Interleaved rounds."""
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
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--full", default="row:32,col:4,r:1@256/0;nnz:64,col:4,r:1@1024/1")
ap.add_argument("--panel", default="row:8,col:4,r:1@256/4")
ap.add_argument("--pw", type=int, default=128)
ap.add_argument("--rounds", type=int, default=5)
args = ap.parse_args()
dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(4, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
del g
rp = a.row_ptr.cpu().numpy().astype(np.int64)
n, pw = args.n, args.pw
b = bench.dense_b(a.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)


def cand(text):
    pt, rest = text.split("@")
    p, v = rest.split("/")
    return Candidate(pt, int(p), 0, int(v))


arms = []
for text in args.full.split(";"):
    cd = cand(text)
    k = plan_for(cd, n, a.num_rows, a.num_cols, rp)
    arms.append((f"N={n} {text}", [(k, prepare_aux(k, a), b, c, cd.hw_variant)]))
cd = cand(args.panel)
kp = plan_for(cd, pw, a.num_rows, a.num_cols, rp)
auxp = prepare_aux(kp, a)
bs = [b[:, i:i + pw].contiguous() for i in range(0, n, pw)]
cs = [torch.empty((a.num_rows, pw), dtype=torch.float32, device=dev) for _ in bs]
arms.append((f"{n // pw}x{pw} {args.panel}", [(kp, auxp, bi, ci, cd.hw_variant) for bi, ci in zip(bs, cs)]))
stream = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _, calls in arms:
    for k, ax, bi, ci, v in calls:
        spmm(k, a, bi, ci, aux=ax, hw_variant=v)
torch.cuda.synchronize()
print("panels equal the full-width result:",
      float((torch.cat(cs, dim=1) - c).abs().max()), flush=True)
res = {name: [] for name, _ in arms}
for _ in range(args.rounds):
    for name, calls in arms:
        ts = []
        for _ in range(3):
            e0.record(stream)
            for k, ax, bi, ci, v in calls:
                spmm(k, a, bi, ci, aux=ax, hw_variant=v)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name].append(statistics.median(ts))
print(desc, "N", n)
base = statistics.median(res[arms[0][0]])
for name in res:
    m = statistics.median(res[name])
    print(f"{name:44s} median {m:.3f} ms ({m / base:.3f}x)  rounds "
          + " ".join(f"{x:.2f}" for x in res[name]), flush=True)
