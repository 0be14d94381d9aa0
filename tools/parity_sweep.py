"""Parity of EVERY schedule candidate (every templated point of the B200 knob
grid x every applicable walk variant) on a BASELINE workload against the
float64 oracle, metric max|got-want|/(|want|+1) (runner.py:159-162), bound
1e-5 (BASELINE.json north star).

The reference product is computed once on the device by
sgap_reference_spmm_f64 (the oracle's arithmetic, matrices.py:241-254) and
pinned bit-for-bit against the CPU oracle (oracle/spmm_oracle.c) on a sample
of rows, so each candidate's check is a device-side reduction.

    python tools/parity_sweep.py --config 3 --out profiles/r01_parity_cfg3.json
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import oracle  # noqa: E402
from paper_2209_02882_b200 import _native  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, reference_spmm_f64, spmm  # noqa: E402
from paper_2209_02882_b200.selector import candidates, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--tol", type=float, default=1e-5)
ap.add_argument("--out", default="")
ap.add_argument("--sample-rows", type=int, default=2000)
ap.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                help="f64: the reference's default precision (sim.run precision='double')")
args = ap.parse_args()

dev = torch.device("cuda", 0)
n = args.n or bench.default_n(args.config)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
dt = torch.float64 if args.dtype == "f64" else torch.float32
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(dt))
b = bench.dense_b(g.num_cols, n, 1, dev).to(dt)
c = torch.empty((a.num_rows, n), dtype=dt, device=dev)
rp = a.row_ptr.cpu().numpy().astype(np.int64)
want = reference_spmm_f64(a, b, n)

# pin the device reference to the CPU oracle on a row sample (incl. the longest rows)
rng = np.random.default_rng(7)
lens = np.diff(rp)
rows = np.unique(np.concatenate([rng.integers(0, a.num_rows, args.sample_rows),
                                 np.argsort(lens)[-64:]]))
ci = a.col_idx.cpu().numpy()
av = a.vals.cpu().numpy()
sub_rp = np.concatenate([[0], np.cumsum(lens[rows])]).astype(np.int32)
sub_ci = np.concatenate([ci[rp[r]:rp[r + 1]] for r in rows]).astype(np.int32)
sub_av = np.concatenate([av[rp[r]:rp[r + 1]] for r in rows])
cpu = oracle.spmm_f64(sub_rp, sub_ci, sub_av, b.cpu().numpy(), n)
dev_rows = want[torch.as_tensor(rows, device=dev)].cpu().numpy()
pinned = bool(np.array_equal(cpu.reshape(dev_rows.shape), dev_rows))
print(desc, f"N={n}", "device reference == CPU oracle on", len(rows), "rows:", pinned, flush=True)


def max_rel_error() -> float:
    err = 0.0
    step = max(1, (1 << 27) // max(n, 1))
    for r0 in range(0, a.num_rows, step):
        w = want[r0:r0 + step]
        e = ((c[r0:r0 + step].double() - w).abs() / (w.abs() + 1.0)).max()
        err = max(err, float(e.item()))
    return err


rows_out, fails = [], []
t0 = time.time()
for cand in candidates(n):
    k = plan_for(cand, n, a.num_rows, a.num_cols, rp)
    if k is None:
        continue
    aux = prepare_aux(k, a, row_ptr_host=rp)
    c.fill_(float("nan"))
    try:
        spmm(k, a, b, c, aux=aux, hw_block=cand.hw_block, hw_variant=cand.hw_variant)
    except _native.SgapError as e:
        if e.status != _native.ERR_ARG:
            raise
        continue
    err = max_rel_error()
    rows_out.append({"cand": cand.label(), "family": k.family, "err": err})
    if not err <= args.tol:
        fails.append(rows_out[-1])
        print("FAIL", cand.label(), err, flush=True)
    del aux
summary = {"workload": desc, "n": n, "dtype": args.dtype, "candidates": len(rows_out), "tol": args.tol,
           "failures": len(fails), "max_err": max(r["err"] for r in rows_out),
           "worst": max(rows_out, key=lambda r: r["err"]), "device_reference_pinned": pinned,
           "seconds": time.time() - t0}
print(json.dumps(summary, indent=1))
if args.out:
    Path(args.out).write_text(json.dumps({"summary": summary, "fails": fails, "rows": rows_out},
                                         indent=1) + "\n")
