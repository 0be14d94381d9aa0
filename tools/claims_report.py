"""Render profiles/r02_paper_claims.md from the measured JSON
(tools/paper_claims.py on configs 2-4, tools/dgsparse_grid.py)."""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
claims = json.loads((ROOT / "profiles" / "r02_paper_claims_cfg234.json").read_text())
grid = json.loads((ROOT / "profiles" / "r02_dgsparse_grid.json").read_text())
out = ["# Paper claims on the BASELINE configs (round 2, one B200)", "",
       "Measured with `tools/paper_claims.py --matrices cfg2,cfg3,cfg4 --n 4,16,64,128` and "
       "`tools/dgsparse_grid.py` (float32, device-resident operands, best of 3-5 launches, zero-fill "
       "included).  Speed-up = time(baseline) / time(Sgap schedule); > 1 means the paper's side wins.",
       "", "## Flexible group size and segment groups (PAPER.md:357-395)", "",
       "| matrix | N | flex r=4 vs r=32 | flex r=8 vs r=32 | segment r=8 vs best row-group | segment r=32 vs best row-group | best Sgap schedule (ms) | vs best DA-SpMM corner |",
       "|---|---|---|---|---|---|---|---|"]
for rec in claims:
    c = rec["claims"]
    f = lambda k: f"{c[k]['speedup']:.2f}" if k in c else "-"  # noqa: E731
    best = c["best_vs_da_spmm"]
    out.append(f"| {rec['matrix']} | {rec['n']} | {f('flex_r4_vs_r32')} | {f('flex_r8_vs_r32')} | "
               f"{f('segment_r8_vs_best_rowgroup')} | {f('segment_r32_vs_best_rowgroup')} | "
               f"`{best['best'][0]}` {best['best'][1]:.3f} | {best['speedup_vs_best_corner']:.2f} |")
out += ["", "Paper (RTX 2080/3090/V100, SuiteSparse, N=4): flexible r=8 vs r=32 2.09-2.45x; segment "
        "vs best row-group 1.01-1.38x; new Sgap algorithms vs TACO 1.10-1.22x.", "",
        "## dgSPARSE RB+PR+RM fine-grained tuning (PAPER.md:408-467)", "",
        "Every cell <groupSz, blockSz, tileSz, workerDimR scale> of `space.enumerate_fine_grained` "
        "executed by `k_rbpr_grid` (`sgap_run_rbpr_grid`); default = dgSPARSE's <32,256,32,1>.  "
        "Default and best cell of each case checked against the float64 reference (<= 1e-5).", "",
        "| matrix | N | cells | default ms | best cell | best ms | tuned / default |",
        "|---|---|---|---|---|---|---|"]
for r in grid["results"]:
    out.append(f"| {r['label']} | {r['n']} | {r['cells']} | {r['default_ms']:.3f} | `{r['best_cell']}` | "
               f"{r['best_ms']:.3f} | {r['tuned_vs_default']:.2f}x |")
out += ["", "| N | tuned vs default, geomean (max) | best static cell | dynamic vs static, geomean | paper (RTX 3090 / 2080 / V100) |",
        "|---|---|---|---|---|"]
paper = {"4": ("2.05 / 2.31 / 1.85", "1.41 / 1.31 / 1.33"), "16": ("2.00 / 2.00 / 1.69", "1.31 / 1.28 / 1.37"),
         "64": ("2.18 / 1.93 / 1.82", "1.11 / 1.11 / 1.18"), "128": ("2.30 / 1.94 / 1.87", "1.12 / 1.10 / 1.14")}
for n, s in grid["summary"].items():
    p = paper.get(str(n), ("-", "-"))
    out.append(f"| {n} | {s['tuned_vs_default_geomean']:.2f} ({s['tuned_vs_default_max']:.2f}) | "
               f"`{s['best_static']}` | {s['dynamic_vs_static_geomean']:.2f} | tuned {p[0]}; dynamic {p[1]} |")
out += ["", "Segment groups are timed with both hardware mappings of the nnz-one family (the shuffle scan and the serial segment walk, hw variants 0/1) and the faster one is reported.  ", "",
        "Reading: on B200 the tuned grid beats dgSPARSE's default cell by more than on the paper's "
        "GPUs at large N (the default gives every 4-column vector of a row its own 32-lane warp, so wide "
        "B rows are gathered 16 bytes per lane), and by about the paper's margin at N = 4-16; a per-"
        "matrix choice beats the best single static cell by 1.25-1.75x, i.e. at or above the paper's "
        "1.1-1.4x.  Power-law matrices (R-MAT, Chung-Lu, configs 2/3) gain least at N = 4: their hub "
        "rows want the 32-lane groups the default already has."]
(ROOT / "profiles" / "r02_paper_claims.md").write_text("\n".join(out) + "\n")
print("\n".join(out))
