"""Shifted-block RB walk (row-multiple hw variants 8 / 9) against the
warp-per-row walk (variant 4) on the BASELINE stencil (config 4): bitwise
equality of C, max_rel_error against the CPU oracle, interleaved timings."""
import argparse
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--ns", default="128,256")
ap.add_argument("--points", default="row:8,col:4,r:1@256;row:4,col:4,r:1@256")
ap.add_argument("--variants", default="4,8,9")
ap.add_argument("--blocks", default="0,128")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--check", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
rp = a.row_ptr.cpu().numpy().astype(np.int64)
print(desc, "nnz", a.nnz)
for n in [int(x) for x in args.ns.split(",")]:
    b = bench.dense_b(g.num_cols, n, 1, dev)
    c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
    cands = []
    for item in args.points.split(";"):
        pt, p = item.split("@")
        for hv in args.variants.split(","):
            for hb in args.blocks.split(","):
                cands.append(Candidate(pt, int(p), int(hb), int(hv)))
    plans = []
    ref = None
    for cd in cands:
        k = plan_for(cd, n, a.num_rows, a.num_cols, rp)
        aux = prepare_aux(k, a)
        try:
            spmm(k, a, b, c, aux=aux, hw_block=cd.hw_block, hw_variant=cd.hw_variant)
        except Exception as e:  # variant not applicable here
            print(f"n={n} {cd.label():34s} refused: {e}", flush=True)
            continue
        torch.cuda.synchronize()
        out = c.clone()
        if ref is None:
            ref = out
        same = bool(torch.equal(out, ref))
        plans.append((cd, k, aux))
        print(f"n={n} {cd.label():34s} bitwise-equal-to-first {same}", flush=True)
    if args.check:
        import oracle
        want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(), a.vals.cpu().numpy(),
                               b.cpu().numpy(), n)
        print(f"n={n} max_rel_error {oracle.max_rel_error(ref.cpu().numpy(), want):.3e}")
    times = {cd.label(): [] for cd, _, _ in plans}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rnd in range(args.rounds):
        order = plans if rnd % 2 == 0 else plans[::-1]
        for cd, k, aux in order:
            best = float("inf")
            for _ in range(3):
                e0.record()
                spmm(k, a, b, c, aux=aux, hw_block=cd.hw_block, hw_variant=cd.hw_variant)
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            times[cd.label()].append(best)
    base = statistics.median(times[plans[0][0].label()])
    for lab, ts in sorted(times.items(), key=lambda kv: statistics.median(kv[1])):
        m = statistics.median(ts)
        print(f"n={n} {lab:34s} {m:8.3f} ms  {m / base:6.3f}x of first  "
              f"{2.0 * a.nnz * n / (m * 1e6):8.1f} GF/s", flush=True)
    del b, c, ref
    torch.cuda.empty_cache()
