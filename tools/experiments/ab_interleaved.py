"""Interleaved A/B of walk variants on one workload: rounds of (v_a, v_b, ...)
each timed as the median of --reps launches, so clock / power drift hits all
variants alike.  Also times the probe-style hint (exactly the top-H columns
by argsort) next to the planner's threshold hint when --probe-h is given."""
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
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--point", default="nnz:512,col:4,r:1")
ap.add_argument("--variants", default="1,9,5")
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--probe-h", type=int, default=0)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--hints", action="store_true", help="force the planner's cold-column hints")
args = ap.parse_args()
dev = torch.device("cuda", 0)
n = args.n or bench.default_n(args.config)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
del g
torch.cuda.empty_cache()
b = bench.dense_b(a.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
rp = a.row_ptr.cpu().numpy().astype(np.int64)
from paper_2209_02882_b200.selector import _first_p  # noqa: E402
k = plan_for(Candidate(args.point, _first_p(args.point, n)), n, a.num_rows, a.num_cols, rp)
aux = prepare_aux(k, a, l2_hints=True if args.hints else None)
arms = [(f"v{v}", a, aux, int(v)) for v in args.variants.split(",")]
if args.probe_h:
    counts = torch.bincount(a.col_idx.long(), minlength=a.num_cols)
    order = torch.argsort(counts, descending=True)
    hot = torch.zeros(a.num_cols, dtype=torch.bool, device=dev)
    hot[order[:args.probe_h]] = True
    col2 = a.col_idx | ((~hot[a.col_idx.long()]).to(torch.int32) << 31)
    a2 = DeviceCsr(a.num_rows, a.num_cols, a.row_ptr, col2, a.vals)
    aux2 = prepare_aux(k, a2, l2_hints=False)
    # the probe form: flagged indices in col_idx itself, read by variant 9's
    # walk through the plan's pointer -- reuse variant 9 with a plan whose
    # hinted copy IS the flagged array
    aux2.plan.aux.d_col_hinted = col2.data_ptr()
    arms.append((f"probe-H{args.probe_h}", a2, aux2, 9))
    th = int(counts[order[args.probe_h - 1]].item())
    print("probe H", args.probe_h, "threshold count", th, "ties at threshold",
          int((counts == th).sum().item()), flush=True)
stream = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {name: [] for name, *_ in arms}
for name, aa, ax, v in arms:
    spmm(k, aa, b, c, aux=ax, hw_variant=v)
for _ in range(args.rounds):
    for name, aa, ax, v in arms:
        ts = []
        for _ in range(args.reps):
            e0.record(stream)
            spmm(k, aa, b, c, aux=ax, hw_variant=v)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name].append(statistics.median(ts))
print(desc, args.point)
base = statistics.median(res[arms[0][0]])
for name in res:
    m = statistics.median(res[name])
    print(f"{name:16s} median {m:.3f} ms ({m / base:.3f}x of {arms[0][0]})  rounds "
          + " ".join(f"{x:.2f}" for x in res[name]), flush=True)
