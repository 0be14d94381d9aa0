"""The reference compiler's own kernels vs this engine, schedule by schedule,
on the B200 (baseline/refgen).

For each frozen reference kernel at the config's dense width, time
  ref  -- the emitted text compiled for sm_100a (float32 instantiation, C
          zero-fill + kernel, the reference's launch geometry), and
  ours -- sgap_run for the same point (float32, every walk variant the
          point admits, best of them), and check both against the oracle.
Times: best of --reps, CUDA events.  Writes a JSON table (--out) and prints
a summary: per-point speed-ups, geomean, best-vs-best, DA-SpMM corners.

    python tools/refgen_bench.py --config 1 --out profiles/r01_refgen_cfg1.json
"""
from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import oracle  # noqa: E402
from baseline import refgen  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, device_block_starts, prepare_aux, spmm  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--max-ms", type=float, default=200.0, help="skip repeats of slower kernels")
ap.add_argument("--out", default="")
args = ap.parse_args()

dev = torch.device("cuda", 0)
n = {1: 32, 2: 128}[args.config]
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(torch.float32))
b = bench.dense_b(g.num_cols, n, 1, dev)
c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
rp = a.row_ptr.cpu().numpy().astype(np.int64)
want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(), a.vals.cpu().numpy(),
                       b.cpu().numpy(), n)
flops = 2.0 * a.nnz * n
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn) -> float:
    fn()
    best = float("inf")
    for _ in range(args.reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
        if best > args.max_ms:
            break
    return best


def err() -> float:
    return float(oracle.max_rel_error(c.cpu().numpy(), want))


rows = []
for rk in refgen.kernels():
    if rk.n != n:
        continue
    k = plan_for(Candidate(rk.point, rk.p), n, a.num_rows, a.num_cols, rp)
    starts = device_block_starts(a, k.chunk, k.grid_size) if rk.has_block_starts else None
    t_ref = timed(lambda: refgen.run(rk, k.grid_size, a, b, c, starts))
    e_ref = err()
    aux = prepare_aux(k, a)
    variants = [0]
    if k.family == "nnz-multiple":
        variants = [1, 2] + ([3, 4] if n // k.c >= 32 else [])
    elif k.family == "row-multiple" and n // k.c <= 256:
        variants = [0, 2]
    best_v, t_ours = None, float("inf")
    for v in variants:
        try:
            t = timed(lambda: spmm(k, a, b, c, aux=aux, hw_variant=v))
        except Exception:  # variant not applicable (e.g. TMA alignment)
            continue
        if t < t_ours:
            best_v, t_ours = v, t
    spmm(k, a, b, c, aux=aux, hw_variant=best_v)
    e_ours = err()
    rows.append({"point": rk.point, "p": rk.p, "family": rk.family, "corner": rk.da_spmm_corner,
                 "ref_ms": t_ref, "ref_err": e_ref, "ours_ms": t_ours, "ours_variant": best_v,
                 "ours_err": e_ours, "speedup": t_ref / t_ours})
    print(f"{rk.point:24s} p{rk.p:<5d} ref {t_ref:9.3f} ms ({e_ref:.1e})  ours {t_ours:8.3f} ms "
          f"v{best_v} ({e_ours:.1e})  x{t_ref / t_ours:7.2f}", flush=True)

sp = [r["speedup"] for r in rows]
best_ref = min(rows, key=lambda r: r["ref_ms"])
best_ours = min(rows, key=lambda r: r["ours_ms"])
summary = {
    "workload": desc, "n": n, "nnz": a.nnz, "points": len(rows),
    "geomean_speedup": math.exp(sum(math.log(s) for s in sp) / len(sp)),
    "min_speedup": min(sp), "max_speedup": max(sp),
    "best_ref": {"point": best_ref["point"], "ms": best_ref["ref_ms"],
                 "gflops": flops / best_ref["ref_ms"] / 1e6},
    "best_ours": {"point": best_ours["point"], "ms": best_ours["ours_ms"],
                  "gflops": flops / best_ours["ours_ms"] / 1e6},
    "best_vs_best": best_ref["ref_ms"] / best_ours["ours_ms"],
    "corners": {r["point"]: {"ref_ms": r["ref_ms"], "ours_ms": r["ours_ms"]}
                for r in rows if r["corner"]},
    "max_ref_err": max(r["ref_err"] for r in rows), "max_ours_err": max(r["ours_err"] for r in rows),
}
print(json.dumps(summary, indent=1))
if args.out:
    Path(args.out).write_text(json.dumps({"summary": summary, "rows": rows}, indent=1) + "\n")
