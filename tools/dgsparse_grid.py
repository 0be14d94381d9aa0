"""Execute the dgSPARSE RB+PR+RM fine-grained tuning grid on B200 (PAPER.md:
408-467; the cells of space.enumerate_fine_grained, which the reference only
enumerates) and reproduce the paper's two tables:

  * tuned vs original: per (matrix, N) the best cell over the default
    dgSPARSE cell <groupSz=32, blockSz=256, tileSz=32, workerDimR=M>
    (PAPER.md tab-over-ori: geomean 1.6-2.3x on RTX 3090/2080/V100);
  * dynamic vs static: per N the single best cell across matrices ("best
    static") against each matrix's own best (tab-over-static: 1.1-1.4x).

Every cell runs ``sgap_run_rbpr_grid`` (k_rbpr_grid) on device-resident
operands; best of --reps launches.  The default and best cells of each case
are checked against the float64 device reference (<= 1e-5).

    python tools/dgsparse_grid.py --out gpurun_out/dgsparse.json
"""
import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2209_02882_b200 import _native  # noqa: E402
from paper_2209_02882_b200 import generators as G  # noqa: E402
from paper_2209_02882_b200.device import (DeviceCsr, prepare_aux, reference_spmm_f64,  # noqa: E402
                                          spmm_rbpr_grid)
from paper_2209_02882_b200.lowering import KernelConfig, lower  # noqa: E402
from paper_2209_02882_b200.selector import _first_p  # noqa: E402
from paper_2209_02882_b200.space import enumerate_fine_grained, parse_point  # noqa: E402
from paper_2209_02882_b200.templates import algorithm_template  # noqa: E402


class _Rp:
    def __init__(self, m, k, rp):
        self.num_rows, self.num_cols, self.row_ptr = m, k, rp


def matrices(dev, which):
    table = {
        "cfg1": lambda: ("config 1: uniform 4096^2 1%", G.config_matrix(1, device=dev)),
        "cfg2": lambda: ("config 2: R-MAT scale 20", G.config_matrix(2, device=dev)),
        "cfg3": lambda: ("config 3: Reddit-shaped", G.config_matrix(3, device=dev)),
        "cfg4": lambda: ("config 4: 27-pt stencil 160^3", G.config_matrix(4, device=dev)),
        "rmat18": lambda: ("R-MAT scale 18", G.rmat(18, 16, seed=1, device=dev)),
        "stencil64": lambda: ("27-pt stencil 64^3", G.stencil27(64, device=dev)),
        "chunglu": lambda: ("Chung-Lu 100k x 10M", G.chung_lu(100_000, 1e7, seed=1, device=dev)),
    }
    for key in which:
        yield key, *table[key]()


def cell_key(c) -> str:
    return f"<{c.group_size},{c.block_size},{c.tile_size},{c.worker_scale}>"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--matrices", default="cfg1,rmat18,stencil64,chunglu,cfg2,cfg3,cfg4")
    ap.add_argument("--ns", default="4,16,64,128")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    for key, label, g in matrices(dev, args.matrices.split(",")):
        a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
                      g.vals.to(torch.float32))
        del g
        rp = a.row_ptr.cpu().numpy().astype(np.int64)
        for n in [int(x) for x in args.ns.split(",")]:
            gen = torch.Generator(device=dev)
            gen.manual_seed(2)
            b = torch.rand((a.num_cols, n), generator=gen, device=dev) * 2 - 1
            c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
            plans = {}
            times = {}
            t_start = time.time()
            for cell in enumerate_fine_grained(n):
                gsz, cz = cell.group_size, cell.coarsen_size
                if gsz not in plans:
                    text = f"row:1/{gsz},col:{cz},r:{gsz}"
                    p = _first_p(text, n)
                    tpl = algorithm_template(parse_point(text), KernelConfig(n=n, p=p))
                    k = lower(tpl, _Rp(a.num_rows, a.num_cols, rp), compute_starts=False)
                    plans[gsz] = (k, prepare_aux(k, a))
                k, aux = plans[gsz]
                kw = dict(block=cell.block_size, tile=cell.tile_size,
                          worker_scale=float(cell.worker_scale), aux=aux, stream=stream)
                try:
                    spmm_rbpr_grid(k, a, b, c, **kw)
                except _native.SgapError as e:
                    if e.status == _native.ERR_CONFIG:
                        continue  # > 1024 threads per block: not launchable
                    raise
                best = math.inf
                for _ in range(args.reps):
                    ev0.record(stream)
                    spmm_rbpr_grid(k, a, b, c, **kw)
                    ev1.record(stream)
                    ev1.synchronize()
                    best = min(best, ev0.elapsed_time(ev1))
                times[cell_key(cell)] = (best, cell)
            default = next(v for kk, v in times.items()
                           if kk == "<32,256,32,1>")
            best_key = min(times, key=lambda kk: times[kk][0])
            want = reference_spmm_f64(a, b, n)
            errs = {}
            for kk in ("<32,256,32,1>", best_key):
                cell = times[kk][1]
                k, aux = plans[cell.group_size]
                c.fill_(float("nan"))
                spmm_rbpr_grid(k, a, b, c, block=cell.block_size, tile=cell.tile_size,
                               worker_scale=float(cell.worker_scale), aux=aux, stream=stream)
                errs[kk] = float(((c.double() - want).abs() / (want.abs() + 1)).max().item())
                assert errs[kk] <= 1e-5, (key, n, kk, errs[kk])
            del want
            rec = {"matrix": key, "label": label, "n": n, "nnz": a.nnz, "cells": len(times),
                   "default_ms": default[0], "best_cell": best_key, "best_ms": times[best_key][0],
                   "tuned_vs_default": default[0] / times[best_key][0], "errors": errs,
                   "times": {kk: v[0] for kk, v in times.items()},
                   "sweep_s": time.time() - t_start}
            results.append(rec)
            print(f"{key} N={n}: default {default[0]:.3f} ms, best {best_key} "
                  f"{times[best_key][0]:.3f} ms -> {rec['tuned_vs_default']:.2f}x "
                  f"({len(times)} cells, {rec['sweep_s']:.0f}s)", flush=True)
            del b, c
        del a
        torch.cuda.empty_cache()
    # tables
    summary = {}
    for n in sorted({r["n"] for r in results}):
        rs = [r for r in results if r["n"] == n]
        gm = math.exp(sum(math.log(r["tuned_vs_default"]) for r in rs) / len(rs))
        common = set.intersection(*[set(r["times"]) for r in rs])
        # best static: the cell minimising the geomean time ratio to each matrix's best
        def score(kk):
            return sum(math.log(r["times"][kk] / r["best_ms"]) for r in rs)
        static = min(common, key=score)
        dyn = math.exp(score(static) / len(rs))
        summary[n] = {"tuned_vs_default_geomean": gm,
                      "tuned_vs_default_max": max(r["tuned_vs_default"] for r in rs),
                      "best_static": static, "dynamic_vs_static_geomean": dyn,
                      "matrices": len(rs)}
        print(f"N={n}: tuned vs default geomean {gm:.3f} (max {summary[n]['tuned_vs_default_max']:.2f}); "
              f"best static {static}, dynamic vs static {dyn:.3f}", flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps({"results": results, "summary": summary}, indent=1))


if __name__ == "__main__":
    main()
