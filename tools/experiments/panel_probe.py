"""Column-panel probe: is one SpMM at width N slower than N/P SpMMs at width
P over contiguous column panels of B and C?  Each panel's B rows are a
smaller L2 working set (K x P x 4 bytes), at the cost of re-reading A once
per panel.  The panels here are separate contiguous arrays (the cheapest
faithful stand-in for a strided panel walk: same sectors per gather, same
L2 footprint per pass).  Interleaved rounds, median of --reps per arm."""
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
from paper_2209_02882_b200.selector import Candidate, _first_p, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--panels", default="128,64,32")
ap.add_argument("--point", default="nnz:512,col:4,r:1")
ap.add_argument("--variant", type=int, default=1)
ap.add_argument("--panel-variant", type=int, default=-1)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
del g
torch.cuda.empty_cache()
rp = a.row_ptr.cpu().numpy().astype(np.int64)
n = args.n
b = bench.dense_b(a.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)


def plan(width):
    k = plan_for(Candidate(args.point, _first_p(args.point, width)), width, a.num_rows,
                 a.num_cols, rp)
    return k, prepare_aux(k, a)


arms = []
k_full, aux_full = plan(n)
arms.append((f"N={n}", [(k_full, aux_full, b, c, args.variant)]))
if aux_full.plan.aux.panel_lanes:  # the in-library column-panel walk (hw variant 10)
    arms.append((f"v10/{aux_full.plan.aux.panel_lanes * k_full.c}", [(k_full, aux_full, b, c, 10)]))
cp = {}
for p in (int(x) for x in args.panels.split(",")):
    if n % p or p >= n:
        continue
    kp, auxp = plan(p)
    bs = [b[:, i:i + p].contiguous() for i in range(0, n, p)]
    cs = [torch.empty((a.num_rows, p), dtype=torch.float32, device=dev) for _ in bs]
    pv = args.panel_variant if args.panel_variant >= 0 else args.variant
    arms.append((f"{n // p}x{p}", [(kp, auxp, bi, ci, pv) for bi, ci in zip(bs, cs)]))
    cp[arms[-1][0]] = cs
    # the same with the panels re-cut from B on every call (what variant 10
    # pays in k_panelize)
    arms.append((f"{n // p}x{p}+cut", [("cut", b, bs, p)] +
                 [(kp, auxp, bi, ci, pv) for bi, ci in zip(bs, cs)]))
stream = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {name: [] for name, _ in arms}
for name, calls in arms:
    for call in calls:
        if call[0] != "cut":
            k, ax, bi, ci, v = call
            spmm(k, a, bi, ci, aux=ax, hw_variant=v)
# panels must reproduce the full-width result bit for bit
torch.cuda.synchronize()
for name, cs in cp.items():
    same = torch.equal(torch.cat(cs, dim=1), c)
    print(name, "bit-identical to the full-width result:", same, flush=True)
for _ in range(args.rounds):
    for name, calls in arms:
        ts = []
        for _ in range(args.reps):
            e0.record(stream)
            for call in calls:
                if call[0] == "cut":
                    for j, bj in enumerate(call[2]):
                        bj.copy_(call[1][:, j * call[3]:(j + 1) * call[3]])
                    continue
                k, ax, bi, ci, v = call
                spmm(k, a, bi, ci, aux=ax, hw_variant=v)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name].append(statistics.median(ts))
print(desc, args.point, "variant", args.variant)
base = statistics.median(res[arms[0][0]])
for name in res:
    m = statistics.median(res[name])
    print(f"{name:10s} median {m:.3f} ms ({m / base:.3f}x)  rounds "
          + " ".join(f"{x:.2f}" for x in res[name]), flush=True)
