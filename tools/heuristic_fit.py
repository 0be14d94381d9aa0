"""Score selector.heuristic offline against the exhaustive device sweeps
stored by tools/selector_regret.py (profiles/r02_selector_regret_full.json:
every candidate's time per matrix x N): regret = time(pick) / time(best),
the pick's time looked up by its point and variant (any p when its own p was
not swept)."""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2209_02882_b200.selector import MatrixStats, heuristic  # noqa: E402


def lookup(times: dict, label: str):
    """The pick's time: the same point and hardware variant at any p (the
    hardware kernels do not depend on p -- it only sizes the reference's
    logical blocks -- so differences between p are sweep noise)."""
    point = label.split("@")[0]
    var = label.split("/v")[1] if "/v" in label else None
    alts = [t for k, t in times.items() if k.split("@")[0] == point and
            ((k.split("/v")[1] if "/v" in k else None) == var)]
    return min(alts) if alts else None


def score(path=ROOT / "profiles" / "r02_selector_regret_full.json", verbose=True):
    rows = json.loads(Path(path).read_text())
    regs = []
    for r in rows:
        st = MatrixStats(**r["stats"])
        h = heuristic(st, r["n"])
        t = lookup(r["times"], h.label())
        best = min(r["times"].values())
        reg = t / best if t else float("nan")
        regs.append(reg)
        if verbose:
            print(f"{r['matrix']:24s} n={r['n']:4d} pick {h.label():34s} regret {reg:.3f}  "
                  f"best {min(r['times'], key=r['times'].get)}")
    ok = [x for x in regs if x == x]
    gm = math.exp(sum(math.log(x) for x in ok) / len(ok))
    print(f"geomean regret {gm:.3f} over {len(ok)} cases, worst {max(ok):.3f}")
    return gm


if __name__ == "__main__":
    score(sys.argv[1] if len(sys.argv) > 1 else ROOT / "profiles" / "r02_selector_regret_full.json")
