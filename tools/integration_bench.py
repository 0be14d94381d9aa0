"""The reference's own sweep driver (spmmlab.runner.sweep, runner.py:232-260)
over BASELINE config 1 -- every templated point at p = 256 -- with its
executor swapped for the B200 (integration.spmmlab_b200.install), against the
same driver on the reference's simulator for a few points (its per-point
cost is extrapolated; the full simulated sweep takes tens of minutes).
Prints a JSON record.

    python tools/integration_bench.py --sim-points 2 --out gpurun_out/integration.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sim-points", type=int, default=2)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import spmmlab.runner as R
    from spmmlab.space import enumerate_space
    from spmmlab.templates import algorithm_template
    from integration import spmmlab_b200 as I

    cfg = R.KernelConfig(n=32, p=256)
    pts = [p for p in enumerate_space().legal if algorithm_template(p, cfg) is not None]
    mats = [R.resolve_matrix(random_spec=(4096, 4096, 0.01, 1), label="config1")]
    I.install()
    R.sweep(mats, cfg, points=pts[:2], precision="single")  # warm (CUDA context, lazy loading)
    t0 = time.perf_counter()
    rows = R.sweep(mats, cfg, points=pts, precision="single")
    b200_s = time.perf_counter() - t0
    I.uninstall()
    statuses = sorted({r["status"] for r in rows})
    # the simulator on a few of the same points (single core, this host)
    sim = []
    for pt in pts[: args.sim_points]:
        t0 = time.perf_counter()
        r = R.sweep(mats, cfg, points=[pt], precision="single")[0]
        sim.append({"point": str(pt), "seconds": time.perf_counter() - t0, "status": r["status"],
                    "atomic_ops": r["atomic_ops"]})
    per_point_sim = sum(s["seconds"] for s in sim) / len(sim)
    b200_by_point = {r["point"]: r["atomic_ops"] for r in rows}
    rec = {"workload": "config 1: random_csr(4096, 4096, 0.01, seed=1), N=32, p=256",
           "points": len(pts), "statuses": statuses,
           "b200_sweep_seconds": b200_s, "b200_seconds_per_point": b200_s / len(pts),
           "simulator_points": sim, "simulator_seconds_per_point": per_point_sim,
           "simulator_sweep_seconds_extrapolated": per_point_sim * len(pts),
           "speedup_of_the_reference_sweep": per_point_sim * len(pts) / b200_s,
           "atomic_ops_equal_on_sampled_points": all(
               b200_by_point[s["point"]] == s["atomic_ops"] for s in sim)}
    print(json.dumps(rec, indent=1))
    if args.out:
        Path(args.out).write_text(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
