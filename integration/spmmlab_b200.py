"""B200 backend for the reference package ``spmmlab``.

The reference's executor is ``spmmlab.sim.run(kernel, a, b, c0=None, *,
precision="double") -> (DenseMatrix, SimMetrics)`` (``sim.py:431-487``),
called by ``runner.verify_point`` (``runner.py:193``) and through it by
``runner.sweep`` (``runner.py:232-260``), the HTTP service and the CLI.
``install()`` swaps that one function for the B200 engine, so the
reference's own planner (``runner.build_kernel``), oracle check, sweep
schema v1 and callers stay untouched and drive the sm_100a kernels:

    import spmmlab
    from integration.spmmlab_b200 import install
    install()                      # spmmlab.sim.run -> B200 (libsgap.so)
    rows = spmmlab.runner.sweep(matrices, KernelConfig(n=32, p=256))

The returned objects are the reference's own types: a ``DenseMatrix`` of
float64 and a ``SimMetrics`` whose ``atomic_ops`` is counted on the device
(equal to the simulator's, pinned by tests/test_gpu_integration.py) and
whose warp-step counters -- simulator cost units with no GPU meaning -- are
0.  The measured device time of the last call is kept in
``last_device_ms()`` for perf columns.  There is no CPU fallback: without a
GPU and libsgap.so, ``run`` raises.
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

__all__ = ["install", "uninstall", "run", "last_device_ms", "sweep_with_perf"]

_saved: dict = {}
_last = {"device_ms": None}


def run(kernel, a, b, c0=None, *, precision: str = "double"):
    """Drop-in for ``spmmlab.sim.run`` on the B200."""
    import spmmlab.matrices as M
    import spmmlab.sim as S
    from paper_2209_02882_b200.sim import SimulationFault as OurFault
    from paper_2209_02882_b200.sim import run as b200_run

    try:
        out, m = b200_run(kernel, a, b, c0, precision=precision)
    except OurFault as e:  # the reference's exception type, same lane
        raise S.SimulationFault(str(e), lane=e.lane, node=None) from e
    _last["device_ms"] = m.device_ms
    dense = M.DenseMatrix(out.num_rows, out.num_cols, out.vals)
    metrics = S.SimMetrics(max_warp_steps=0, total_steps=0, atomic_ops=int(m.atomic_ops),
                           idle_lane_steps=0)
    return dense, metrics


def last_device_ms():
    return _last["device_ms"]


def install():
    """Route the reference's executor to the B200 (idempotent)."""
    import spmmlab.runner as R
    import spmmlab.sim as S
    if not _saved:
        _saved["sim.run"] = S.run
        _saved["runner.run"] = R.run
    S.run = run
    R.run = run  # runner imported the name (runner.py:28)


def uninstall():
    import spmmlab.runner as R
    import spmmlab.sim as S
    if _saved:
        S.run = _saved.pop("sim.run")
        R.run = _saved.pop("runner.run")


def sweep_with_perf(matrices, config, **kw):
    """``spmmlab.runner.sweep`` rows (frozen schema v1) with the perf columns
    of this engine appended (``device_ms``, ``gflops``)."""
    import spmmlab.runner as R
    install()
    points = kw.pop("points", None)
    if points is None:
        from spmmlab.space import enumerate_space
        points = list(enumerate_space().legal)
    rows = []
    for mi in matrices:
        for pt in points:
            _last["device_ms"] = None
            part = R.sweep([mi], config, points=[pt], **kw)
            for row in part:
                ms = _last["device_ms"] if row.get("status") in ("pass", "fail") else None
                row["device_ms"] = ms
                nnz = mi.matrix.nnz if mi.matrix is not None else 0
                row["gflops"] = (2.0 * nnz * config.n / (ms * 1e6)) if ms else None
            rows.extend(part)
    return rows
