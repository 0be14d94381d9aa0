"""Multi-GPU scaling projected on one B200 (this run has one GPU; the driver
measures the real 1/2/4/8-GPU runs): build exactly the workload
`bench.py --gpus W` builds, time every rank's shard on this GPU (no data-path
collective exists, so a rank's time is its shard's SpMM time),
and report max-over-ranks throughput and efficiency against W x the 1-GPU
value.  Weak scaling = bench's default (R-MAT scale 20 + log2 W, B grows with
the graph); strong = config 5 (R-MAT scale 24, fixed).

    python tools/scaling_projection.py --out profiles/r01_scaling_projection.json
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.partition import plan_shards, shard_csr  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--point", default="nnz:512,col:4,r:1")
ap.add_argument("--variant", type=int, default=1)
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--strong", action="store_true", help="config 5 strong scaling instead")
ap.add_argument("--unpermuted", action="store_true",
                help="strong scaling on the UNPERMUTED R-MAT scale 24 (SURVEY 8(e) stress case)")
ap.add_argument("--balance", default="nnz", choices=["nnz", "bytes", "cost"])
ap.add_argument("--slices", type=int, default=64, help="calibration slices for --balance cost")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default="")
args = ap.parse_args()
dev = torch.device("cuda", 0)
n = 128
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for world in [int(w) for w in args.worlds.split(",")]:
    if args.unpermuted:
        from paper_2209_02882_b200 import generators as G
        g = G.rmat(24, 16, seed=1, permute=False, device=dev)
        desc = f"R-MAT scale 24 unpermuted ({args.balance}-balanced shards)"
    else:
        g, desc, _ = bench.build_workload(5 if args.strong else 2, world, 1, dev,
                                          weak=not args.strong)
    calib = None
    if args.balance == "cost":  # time S nnz-balanced slices alone, cut on their cumulative time
        rph_all = g.row_ptr.cpu().numpy()
        cal_plan = plan_shards(rph_all, args.slices)
        cb = bench.dense_b(g.num_cols, n, 1, dev)
        costs = []
        for sl in range(args.slices):
            rp, ci, vals = shard_csr(g.row_ptr, g.col_idx, g.vals, cal_plan, sl)
            lo, hi = cal_plan.rows(sl)
            a = DeviceCsr(hi - lo, g.num_cols, rp.to(torch.int32).contiguous(),
                          ci.to(torch.int32).contiguous(), vals.to(torch.float32).contiguous())
            rph = a.row_ptr.cpu().numpy().astype(np.int64)
            c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
            k = plan_for(Candidate(args.point, 256), n, a.num_rows, a.num_cols, rph)
            aux = prepare_aux(k, a)
            spmm(k, a, cb, c, aux=aux, hw_variant=args.variant)
            e0.record()
            spmm(k, a, cb, c, aux=aux, hw_variant=args.variant)
            e1.record()
            e1.synchronize()
            costs.append(e0.elapsed_time(e1))
            del a, c, aux, rp, ci, vals
        calib = (cal_plan.starts, np.asarray(costs))
        del cb
    plan = plan_shards(g.row_ptr.cpu().numpy(), world, balance=args.balance, n=n,
                       calibration=calib)
    b = bench.dense_b(g.num_cols, n, 1, dev)
    times = []
    for rank in range(world):
        rp, ci, vals = shard_csr(g.row_ptr, g.col_idx, g.vals, plan, rank)
        lo, hi = plan.rows(rank)
        a = DeviceCsr(hi - lo, g.num_cols, rp.to(torch.int32).contiguous(),
                      ci.to(torch.int32).contiguous(), vals.to(torch.float32).contiguous())
        rph = a.row_ptr.cpu().numpy().astype(np.int64)
        c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
        k = plan_for(Candidate(args.point, 256), n, a.num_rows, a.num_cols, rph)
        aux = prepare_aux(k, a, row_ptr_host=rph)
        spmm(k, a, b, c, aux=aux, hw_variant=args.variant)
        best = float("inf")
        for _ in range(args.reps):
            e0.record()
            spmm(k, a, b, c, aux=aux, hw_variant=args.variant)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        times.append({"rank": rank, "rows": a.num_rows, "nnz": a.nnz, "ms": best})
        del a, c, aux, rp, ci, vals
        torch.cuda.empty_cache()
    t = max(x["ms"] for x in times)
    value = 2.0 * g.nnz * n / (t * 1e6)
    res.append({"world": world, "workload": desc, "nnz": g.nnz, "max_rank_ms": t,
                "shard_rows": [x["rows"] for x in times],
                "gflops": value, "ranks": times})
    print(f"W={world}: {desc}: max-rank {t:.3f} ms -> {value:.0f} GFLOP/s "
          f"(rank ms {min(x['ms'] for x in times):.3f}-{t:.3f})", flush=True)
    del g, b
    torch.cuda.empty_cache()
base = res[0]["gflops"] / res[0]["world"]
for r in res:
    r["efficiency_vs_w1"] = r["gflops"] / (r["world"] * base)
    print(f"W={r['world']}: efficiency {r['efficiency_vs_w1']:.3f}")
if args.out:
    Path(args.out).write_text(json.dumps({"strong": args.strong, "point": args.point,
                                          "projection": res}, indent=1) + "\n")
