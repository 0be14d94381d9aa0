"""Caller integration: the reference's own driver --
``spmmlab.runner.verify_point`` and ``runner.sweep`` from the installed
reference (``baseline/_ref``, pip-installed from /root/reference) -- runs on
the B200 through ``integration.spmmlab_b200.install()``, and this package's
mirror ``runner.sweep`` emits the same frozen schema v1 (+ perf columns).

Skipped where the reference install is absent (it is git-ignored and travels
to the GPU box with the snapshot)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import matrix_zoo
from paper_2209_02882_b200 import runner as ours
from paper_2209_02882_b200.lowering import KernelConfig
from paper_2209_02882_b200.space import parse_point

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def spmmlab():
    if not (REF / "spmmlab").exists():
        pytest.skip("reference install baseline/_ref absent")
    sys.path.insert(0, str(REF))
    import spmmlab  # noqa: F401
    import spmmlab.runner  # noqa: F401
    from integration import spmmlab_b200
    spmmlab_b200.install()
    yield sys.modules["spmmlab"]
    spmmlab_b200.uninstall()


def _ref_matrix(M, mat):
    return M.CsrMatrix(mat.num_rows, mat.num_cols, np.asarray(mat.row_ptr), np.asarray(mat.col_idx),
                       np.asarray(mat.vals))


def test_reference_verify_point_runs_on_b200(spmmlab):
    """The reference's verify_point (its planner, its float64 oracle, its
    error metric) with the B200 executor: every templated point on part of
    the zoo, writebacks equal to the simulator's (tests/golden/sim_metrics.json)."""
    import spmmlab.matrices as M
    import spmmlab.runner as R
    import spmmlab.sim as S
    from integration import spmmlab_b200
    assert R.run is spmmlab_b200.run and S.run is spmmlab_b200.run
    sim = {(r["matrix"], r["n"], r["point"]): r for r in
           json.loads((GOLDEN / "sim_metrics.json").read_text())}
    from spmmlab.space import enumerate_space
    from spmmlab.templates import algorithm_template
    runs = 0
    for n in (4, 8):
        cfg = R.KernelConfig(n=n, p=256)
        pts = [p for p in enumerate_space().legal if algorithm_template(p, cfg) is not None]
        for label, mat, b_seed in matrix_zoo()[::4]:
            a = _ref_matrix(M, mat)
            b = M.random_dense(a.num_cols, n, seed=b_seed)
            for pt in pts:
                for precision, tol in (("double", 1e-12), ("single", 1e-5)):
                    rep = R.verify_point(a, pt, cfg, b=b, precision=precision, tolerance=tol)
                    assert rep.status == "pass", (label, str(pt), precision, rep.max_rel_error)
                    assert isinstance(rep.metrics, S.SimMetrics)
                    assert rep.metrics.atomic_ops == sim[(label, n, str(pt))]["atomic_ops"]
                    runs += 1
    assert runs > 400


def test_reference_sweep_schema_v1_with_perf(spmmlab):
    """runner.sweep of the reference over two matrices (one unreadable) on
    the B200: schema v1 columns, statuses, and the perf columns appended."""
    import spmmlab.runner as R
    from integration.spmmlab_b200 import sweep_with_perf
    mats = [R.resolve_matrix(random_spec=(300, 200, 0.05, 3)),
            R.MatrixInput("broken", None, "unreadable")]
    pts = [parse_point(t) for t in ("nnz:1,col:4,r:8", "row:1/4,col:4,r:4", "nnz:32,col:4,r:1",
                                    "row:2,col:1,r:1", "row:1,col:1/2,r:1")]
    from spmmlab.space import parse_point as ref_parse
    pts = [ref_parse(str(p)) for p in pts]
    rows = R.sweep(mats, R.KernelConfig(n=16, p=256), points=pts)
    assert [r["status"] for r in rows] == ["pass", "pass", "pass", "pass", "no_template",
                                           "matrix_error: unreadable"]
    assert all(tuple(r.keys()) == R.SWEEP_COLUMNS for r in rows)
    csv_text = R.rows_to_csv(rows)
    assert csv_text.splitlines()[0] == ",".join(R.SWEEP_COLUMNS)
    perf = sweep_with_perf(mats[:1], R.KernelConfig(n=16, p=256), points=pts)
    assert [r["status"] for r in perf] == ["pass"] * 4 + ["no_template"]
    assert all(r["device_ms"] and r["gflops"] for r in perf[:4])
    assert perf[4]["device_ms"] is None


def test_reference_fault_maps_to_simulation_fault(spmmlab):
    """An out-of-range column (bypassing CsrMatrix's checks) raises the
    reference's SimulationFault instead of reading out of bounds."""
    import spmmlab.matrices as M
    import spmmlab.runner as R
    import spmmlab.sim as S
    a = M.CsrMatrix(3, 4, [0, 2, 3, 4], [0, 1, 1, 2], [1.0, 2.0, 3.0, 4.0])
    object.__setattr__(a, "col_idx", np.array([0, 9, 1, 2]))  # corrupt after validation
    b = M.random_dense(4, 8, seed=1)
    k = R.build_kernel(R.parse_point("row:1,col:1,r:1"), R.KernelConfig(n=8, p=256), a)
    with pytest.raises(S.SimulationFault):
        S.run(k, a, b)


def test_mirror_sweep_rows(zoo):
    """This package's runner.sweep (a19): frozen schema v1 (+ perf columns),
    no_template and matrix_error rows, csv/json round trip."""
    mats = [ours.MatrixInput(label, mat) for label, mat, _ in zoo[:3]]
    mats.append(ours.MatrixInput("broken", None, "bad header"))
    pts = [parse_point(t) for t in ("nnz:1,col:1,r:4", "row:1/2,col:1,r:2", "nnz:4,col:1,r:1",
                                    "row:1,col:1/2,r:1")]
    rows = ours.sweep(mats, KernelConfig(n=4, p=256), points=pts, precision="single", perf=True)
    assert len(rows) == 3 * 4 + 1
    for r in rows[:-1]:
        assert tuple(r.keys()) == ours.SWEEP_COLUMNS + ours.SWEEP_PERF_COLUMNS
        if str(r["point"]) == "row:1,col:1/2,r:1":
            assert r["status"] == "no_template"
        else:
            assert r["status"] == "pass" and r["device_ms"] > 0
    assert rows[-1]["status"] == "matrix_error: bad header"
    text = ours.rows_to_csv(rows)
    assert text.splitlines()[0].split(",")[-2:] == list(ours.SWEEP_PERF_COLUMNS)
    doc = json.loads(ours.rows_to_json(rows))
    assert doc["schema_version"] == 1 and len(doc["rows"]) == len(rows)
