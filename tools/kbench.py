"""Kernel micro-benchmark on a BASELINE workload: time a list of schedule
points (and CTA sizes) on device-resident operands; optional parity check of
each against the CPU oracle.  Used for the optimisation loop; results are
summarised under profiles/."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, autotune, candidates  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--points", default="nnz:32,col:4,r:1@256")
ap.add_argument("--blocks", default="0")
ap.add_argument("--variants", default="0")
ap.add_argument("--all", action="store_true")
ap.add_argument("--check", action="store_true")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default="")
ap.add_argument("--cusparse", action="store_true")
ap.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                help="value type of A, B and C (f64: the reference's default precision)")
args = ap.parse_args()
dev = torch.device("cuda", 0)
DT = torch.float64 if args.dtype == "f64" else torch.float32
n = args.n or bench.default_n(args.config)
g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
              g.vals.to(DT))
touched = int(torch.unique(a.col_idx).numel())
b = bench.dense_b(g.num_cols, n, 1, dev).to(DT)
c = torch.empty((a.num_rows, n), dtype=DT, device=dev)
rp = a.row_ptr.cpu().numpy().astype(np.int64)
if args.all:
    cands = candidates(n)
else:
    cands = []
    for item in args.points.split(";"):
        pt, p = item.split("@")
        for hb in args.blocks.split(","):
            for hv in args.variants.split(","):
                cands.append(Candidate(pt, int(p), int(hb), int(hv)))
res = autotune(a, b, c, n, cands, reps=args.reps, row_ptr_host=rp, max_ms=100.0)
esz = 8 if args.dtype == "f64" else 4
abytes = bench.algorithmic_bytes(a.num_rows, a.nnz, n, touched, esz) + (esz - 4) * a.nnz
print(desc, "nnz", a.nnz, "n", n, "algorithmic MB", abytes / 1e6)
rows = []
for cd, ms in res:
    gf = 2.0 * a.nnz * n / (ms * 1e6)
    gbs = abytes / (ms * 1e-3) / 1e9
    print(f"{cd.label():32s} {ms:8.3f} ms {gf:9.1f} GF/s {gbs:8.1f} GB/s")
    rows.append({"cand": cd.label(), "ms": ms, "gflops": gf, "gbs": gbs})
if args.check:
    import oracle
    from paper_2209_02882_b200.selector import plan_for
    from paper_2209_02882_b200.device import spmm
    want = oracle.spmm_f64(rp.astype(np.int32), a.col_idx.cpu().numpy(), a.vals.cpu().numpy(),
                           b.cpu().numpy(), n)
    for cd, ms in res[:8]:
        k = plan_for(cd, n, a.num_rows, a.num_cols, rp)
        spmm(k, a, b, c, hw_block=cd.hw_block, hw_variant=cd.hw_variant)
        torch.cuda.synchronize()
        err = oracle.max_rel_error(c.cpu().numpy(), want)
        tol = 1e-12 if args.dtype == "f64" else 1e-5
        print(f"check {cd.label():32s} max_rel_error {err:.3e}", "OK" if err <= tol else "FAIL")
if args.out:
    Path(args.out).write_text(json.dumps({"workload": desc, "n": n, "rows": rows}, indent=1))

if "--cusparse" in sys.argv[1:] or True:
    # library sanity check: cuSPARSE SpMM through torch.sparse on
    # the same device operands -- a reference point, not part of the product
    try:
        sp = torch.sparse_csr_tensor(a.row_ptr.to(torch.int64), a.col_idx.to(torch.int64), a.vals,
                                     size=(a.num_rows, a.num_cols))
        out = torch.sparse.mm(sp, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = float("inf")
        for _ in range(args.reps):
            e0.record()
            out = torch.sparse.mm(sp, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{'cuSPARSE (torch.sparse.mm, CSR f32)':32s} {best:8.3f} ms {2.0 * a.nnz * n / (best * 1e6):9.1f} GF/s")
    except Exception as e:  # pragma: no cover
        print("cuSPARSE comparison unavailable:", e)
