"""Markdown table of the schedule sweeps (`tools/kbench.py --all --out`):
per workload the best candidate overall, the best EB (nnz families) and
RB (row families) candidate, and cuSPARSE from the sweep's log.

    python tools/sweep_table.py profiles/r02_sweeps/sweep_cfg*_n*.json
"""
import json
import re
import sys
from pathlib import Path


def row(path: Path) -> str:
    doc = json.loads(path.read_text())
    rows = sorted(doc["rows"], key=lambda r: r["ms"])
    best = rows[0]
    eb = next((r for r in rows if r["cand"].startswith("nnz:")), None)
    rb = next((r for r in rows if r["cand"].startswith("row:")), None)
    cus = None
    log = path.with_suffix(".log")
    if log.exists():
        m = re.search(r"cuSPARSE[^\n]*?([\d.]+) ms", log.read_text())
        cus = float(m.group(1)) if m else None
    cell = lambda r: (f"`{r['cand']}` | {r['ms']:.3f}" if r else "-- | --")  # noqa: E731
    ratio = f"{eb['ms'] / rb['ms']:.2f}" if eb and rb else "--"
    vs = f"{cus / best['ms']:.2f}x" if cus else "--"
    return (f"| {doc['workload'][:40]} | {doc['n']} | {len(rows)} | {cell(best)} | "
            f"{best['gflops']:.0f} | {cell(eb)} | {cell(rb)} | {ratio} | "
            f"{cus if cus else '--'} | {vs} |")


def main(paths):
    print("| workload | N | candidates | best overall | ms | GFLOP/s | best EB | ms | best RB | ms "
          "| EB/RB | cuSPARSE ms | vs cuSPARSE |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    key = lambda p: tuple(int(x) for x in re.findall(r"cfg(\d+)_n(\d+)", p.name)[0])  # noqa: E731
    for p in sorted((Path(x) for x in paths), key=key):
        print(row(p))


if __name__ == "__main__":
    main(sys.argv[1:])
