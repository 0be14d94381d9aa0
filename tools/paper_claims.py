"""Reproduce the paper's schedule-speedup claims on B200.

For each matrix and dense width N it times, on device-resident operands:

  * flexible group size vs fixed r=32 for {<1/g row, c col>, r=g}
    (r=8 / r=4 vs r=32, 2.1-2.5x on RTX 2080/3090/V100);
  * segment reduction {<1 nnz, c col>, r} vs the best {<1/g row, c col>, g}
    at r = 4/8/16/32 (1.01-1.38x);
  * the best Sgap schedule vs the DA-SpMM fixed corners.

Usage (on the GPU box):  python tools/paper_claims.py --out gpurun_out/claims.json
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2209_02882_b200 import generators as G  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr  # noqa: E402
from paper_2209_02882_b200.lowering import KernelConfig  # noqa: E402
from paper_2209_02882_b200.selector import Candidate, autotune, candidates  # noqa: E402
from paper_2209_02882_b200.space import parse_point  # noqa: E402
from paper_2209_02882_b200.templates import algorithm_template  # noqa: E402


MATRICES = {
    "cfg1": ("config1 uniform 4096^2 1%", lambda dev: G.config_matrix(1, device=dev)),
    "rmat18": ("rmat scale 18 ef 16", lambda dev: G.rmat(18, 16, seed=1, device=dev)),
    "stencil64": ("stencil27 64^3", lambda dev: G.stencil27(64, device=dev)),
    "chunglu": ("chung-lu 100k x ~10M", lambda dev: G.chung_lu(100_000, 1e7, seed=1, device=dev)),
    "cfg2": ("config2 R-MAT scale 20", lambda dev: G.config_matrix(2, device=dev)),
    "cfg3": ("config3 Reddit-shaped", lambda dev: G.config_matrix(3, device=dev)),
    "cfg4": ("config4 stencil27 160^3", lambda dev: G.config_matrix(4, device=dev)),
}


def matrices(dev, keys):
    for k in keys:
        label, make = MATRICES[k]
        yield label, make(dev)


def best_of(a, b, c, n, pts, rp):
    cands = []
    for text in pts:
        for p in (256, 1024):
            if algorithm_template(parse_point(text), KernelConfig(n=n, p=p)) is not None:
                cands.append(Candidate(text, p))
                if text.startswith("nnz:1,"):  # the segment-group family's serial-walk mapping
                    cands.append(Candidate(text, p, 0, 1))
    if not cands:
        return None, None
    res = autotune(a, b, c, n, cands, reps=5, row_ptr_host=rp)
    return res[0][0].point, res[0][1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="4,8")
    ap.add_argument("--matrices", default="cfg1,rmat18,stencil64,chunglu")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = []
    for label, g in matrices(dev, args.matrices.split(",")):
        a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
                      g.vals.to(torch.float32))
        rp = a.row_ptr.cpu().numpy().astype(np.int64)
        for n in (int(x) for x in args.n.split(",")):
            gen = torch.Generator(device=dev)
            gen.manual_seed(2)
            b = torch.rand((a.num_cols, n), generator=gen, device=dev) * 2 - 1
            c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
            rec = {"matrix": label, "nnz": a.nnz, "n": n, "claims": {}}
            cs = [1, 2, 4]
            # 1. flexible r vs fixed r=32, row-reciprocal
            fixed = best_of(a, b, c, n, [f"row:1/32,col:{cc},r:32" if cc > 1 else "row:1/32,col:1,r:32"
                                         for cc in cs], rp)
            for r in (4, 8):
                flex = best_of(a, b, c, n, [f"row:1/{r},col:{cc},r:{r}" if cc > 1 else f"row:1/{r},col:1,r:{r}"
                                            for cc in cs], rp)
                if fixed[1] and flex[1]:
                    rec["claims"][f"flex_r{r}_vs_r32"] = {"fixed": fixed, "flex": flex,
                                                          "speedup": fixed[1] / flex[1]}
            # 2. segment group vs best row group, per r
            for r in (4, 8, 16, 32):
                seg = best_of(a, b, c, n, [f"nnz:1,col:{cc},r:{r}" if cc > 1 else f"nnz:1,col:1,r:{r}"
                                           for cc in cs], rp)
                rowg = best_of(a, b, c, n, [f"row:1/{gg},col:{cc},r:{gg}" if cc > 1 else f"row:1/{gg},col:1,r:{gg}"
                                            for gg in (2, 4, 8, 16, 32) for cc in cs], rp)
                if seg[1] and rowg[1]:
                    rec["claims"][f"segment_r{r}_vs_best_rowgroup"] = {
                        "segment": seg, "rowgroup": rowg, "speedup": rowg[1] / seg[1]}
            # 3. best Sgap schedule vs DA-SpMM fixed corners
            corners = {"EB+SR": "nnz:32,col:1,r:1", "RB+SR": "row:1,col:1,r:1",
                       "RB+PR": "row:1/32,col:1,r:32", "EB+PR": "nnz:1,col:1,r:32"}
            fixed_t = {}
            for name, pt in corners.items():
                bt = best_of(a, b, c, n, [pt], rp)
                if bt[1]:
                    fixed_t[name] = bt
            allc = autotune(a, b, c, n, candidates(n), reps=3, row_ptr_host=rp, max_ms=200.0)
            best = (allc[0][0].label(), allc[0][1])
            rec["claims"]["best_vs_da_spmm"] = {
                "best": best, "corners": fixed_t,
                "speedup_vs_best_corner": min(t for _, t in fixed_t.values()) / best[1],
                "speedup_vs_each": {k: v[1] / best[1] for k, v in fixed_t.items()}}
            print(json.dumps(rec), flush=True)
            out.append(rec)
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
