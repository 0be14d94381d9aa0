"""Regret of selector.heuristic against the exhaustive sweep (SURVEY 8(a)
a20): for each matrix x N, time every candidate of the B200 knob grid and
report time(heuristic pick) / time(best)."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2209_02882_b200 import generators as G  # noqa: E402
from paper_2209_02882_b200.device import DeviceCsr  # noqa: E402
from paper_2209_02882_b200.selector import autotune, candidates, heuristic, matrix_stats  # noqa: E402

CASES = [
    ("config1 uniform", lambda d: G.config_matrix(1, device=d), (4, 32)),
    ("config2 rmat s20", lambda d: G.rmat(20, 16, seed=1, device=d), (8, 128)),
    ("rmat s18", lambda d: G.rmat(18, 16, seed=1, device=d), (4, 32)),
    ("stencil 64^3", lambda d: G.stencil27(64, device=d), (4, 64)),
    ("config4 stencil 160^3", lambda d: G.stencil27(160, device=d), (16, 128)),
    ("chung-lu 100k", lambda d: G.chung_lu(100_000, 1e7, seed=1, device=d), (8, 64)),
    ("config3 reddit-shaped", lambda d: G.config_matrix(3, device=d), (64,)),
]


# matrices the heuristic was NOT fitted on (other sizes, seeds, widths)
HOLDOUT = [
    ("uniform 8192 x 40/row", lambda d: G.uniform_random(8192, 8192, 40.0, seed=7, device=d), (8, 64)),
    ("rmat s19 seed 5", lambda d: G.rmat(19, 16, seed=5, device=d), (4, 16, 128)),
    ("rmat s21 unpermuted", lambda d: G.rmat(21, 8, seed=2, permute=False, device=d), (32, 128)),
    ("stencil 96^3", lambda d: G.stencil27(96, device=d), (8, 32, 256)),
    ("chung-lu 300k", lambda d: G.chung_lu(300_000, 3e7, seed=3, device=d), (16, 128)),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--holdout", action="store_true", help="score on matrices not used for fitting")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows = []
    for label, make, ns in (HOLDOUT if args.holdout else CASES):
        g = make(dev)
        a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
                      g.vals.to(torch.float32))
        del g
        rp = a.row_ptr.cpu().numpy().astype(np.int64)
        st = matrix_stats(rp, a.num_cols)
        for n in ns:
            b = torch.rand((a.num_cols, n), device=dev) * 2 - 1
            c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
            res = autotune(a, b, c, n, candidates(n), reps=2, row_ptr_host=rp, max_ms=60.0)
            h = heuristic(st, n)
            ht = autotune(a, b, c, n, [h], reps=5, row_ptr_host=rp)[0][1]
            best = res[0]
            rec = {"matrix": label, "n": n, "nnz": a.nnz, "stats": st.as_dict(),
                   "best": best[0].label(), "best_ms": best[1], "heuristic": h.label(),
                   "heuristic_ms": ht, "regret": ht / best[1], "candidates": len(res),
                   # every candidate's time, so a revised heuristic can be scored offline
                   "times": {cd.label(): ms for cd, ms in res}}
            print(json.dumps({k: v for k, v in rec.items() if k != "times"}), flush=True)
            rows.append(rec)
            del b, c
        del a
        torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
