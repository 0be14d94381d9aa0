"""GPU parity: every family of sm_100a kernels against the CPU oracle and the
reference's own simulator counters, through the C ABI.

Bars (BASELINE.json north_star / SURVEY 8(c)):
  * float32: max|got - want| / (|want| + 1) <= 1e-5 against the float64 oracle
    fed the same float32-rounded operands;
  * float64: <= 1e-12 against the reference oracle (golden fixture);
  * integers bit-exact: block_starts, grid/block, and the writeback count
    (== SimMetrics.atomic_ops of the reference simulator).
"""

import json

import numpy as np
import pytest
import torch

import oracle
from paper_2209_02882_b200.device import DeviceCsr, device_block_starts
from paper_2209_02882_b200.lowering import KernelConfig, compute_block_starts
from paper_2209_02882_b200.matrices import CsrMatrix, DenseMatrix, random_csr, random_dense
from paper_2209_02882_b200.runner import build_kernel, verify_point
from paper_2209_02882_b200.sim import (SimulationFault, exec_atomic_add_group,
                                       exec_seg_reduce_group, run)
from paper_2209_02882_b200.space import enumerate_space, parse_point
from paper_2209_02882_b200.templates import algorithm_template

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
F64_TOL = 1e-12


def templated(n, p):
    cfg = KernelConfig(n=n, p=p)
    return [pt for pt in enumerate_space().legal if algorithm_template(pt, cfg) is not None]


def oracle_f32(mat, b, n):
    """f64 oracle on the float32-rounded operands (what the device computes on)."""
    return oracle.spmm_f64(np.asarray(mat.row_ptr, np.int32), np.asarray(mat.col_idx, np.int32),
                           np.asarray(mat.vals, np.float32),
                           np.asarray(b.vals, np.float32).reshape(mat.num_cols, n), n)


def test_zoo_every_templated_point_single_and_double(zoo):
    """2 x 66 points x 20 matrices (the reference's acceptance gate 1,
    test_acceptance.py:41-63) in both precisions, plus the simulator's
    writeback counter for each run."""
    sim = {(r["matrix"], r["n"], r["point"]): r for r in
           json.loads((GOLDEN / "sim_metrics.json").read_text())}
    golden = np.load(GOLDEN / "zoo_oracle.npz")
    worst32 = worst64 = 0.0
    runs = 0
    for n in (4, 8):
        cfg = KernelConfig(n=n, p=256)
        pts = templated(n, 256)
        assert len(pts) == 66
        for label, mat, b_seed in zoo:
            b = random_dense(mat.num_cols, n, seed=b_seed)
            want64 = golden[f"{label}|{n}"]
            want32 = oracle_f32(mat, b, n)
            for pt in pts:
                k = build_kernel(pt, cfg, mat)
                got, m = run(k, mat, b, precision="single")
                e32 = oracle.max_rel_error(got.vals, want32)
                assert e32 <= F32_TOL, (label, n, str(pt), e32)
                assert m.atomic_ops == sim[(label, n, str(pt))]["atomic_ops"], (label, n, str(pt))
                got64, m64 = run(k, mat, b, precision="double")
                e64 = oracle.max_rel_error(got64.vals, want64)
                assert e64 <= F64_TOL, (label, n, str(pt), e64)
                assert m64.atomic_ops == m.atomic_ops
                worst32, worst64 = max(worst32, e32), max(worst64, e64)
                runs += 1
    assert runs == 2640
    print(f"zoo: {runs} runs, worst f32 {worst32:.3e}, worst f64 {worst64:.3e}")


@pytest.mark.parametrize("p", [256, 1024])
def test_config1_every_templated_point(p):
    """BASELINE config 1 (4096^2, 1%, N=32): every templated point."""
    a = random_csr(4096, 4096, 0.01, seed=1)
    b = random_dense(4096, 32, seed=2)
    want = oracle_f32(a, b, 32)
    cfg = KernelConfig(n=32, p=p)
    pins = {(s["point"], s["p"]): s for s in json.loads((GOLDEN / "cfg1.json").read_text())["sim"]}
    pts = templated(32, p)
    assert len(pts) == (58 if p == 256 else 66)
    for pt in pts:
        k = build_kernel(pt, cfg, a)
        got, m = run(k, a, b, precision="single")
        err = oracle.max_rel_error(got.vals, want)
        assert err <= F32_TOL, (str(pt), err)
        st = oracle.block_starts(a.row_ptr, k.chunk, k.grid_size) if k.family.startswith("nnz") else None
        wb = oracle.writebacks(k.family, a.row_ptr, 32, k.grid_size, starts=st, npb=k.chunk,
                               r=k.r, chunk=k.chunk, g=k.g)
        assert m.atomic_ops == wb, str(pt)
        if (str(pt), p) in pins:
            assert m.atomic_ops == pins[(str(pt), p)]["atomic_ops"]


@pytest.mark.parametrize("n", [1, 3, 5, 6, 12])
def test_odd_and_narrow_widths_every_templated_point(n):
    """Widths that are not a multiple of 4 take the scalar/float2 tile paths
    (store_vec narrower than 16 B); every templated point, both precisions."""
    a = random_csr(1500, 900, 0.02, seed=11)
    b = random_dense(900, n, seed=12)
    want32 = oracle_f32(a, b, n)
    want64 = oracle.spmm_f64(a.row_ptr, a.col_idx, a.vals, b.vals.reshape(900, n), n)
    cfg = KernelConfig(n=n, p=256)
    pts = templated(n, 256)
    assert pts
    for pt in pts:
        k = build_kernel(pt, cfg, a)
        got, _ = run(k, a, b, precision="single")
        assert oracle.max_rel_error(got.vals, want32) <= F32_TOL, (n, str(pt))
        got64, _ = run(k, a, b, precision="double")
        assert oracle.max_rel_error(got64.vals, want64) <= F64_TOL, (n, str(pt))


def test_device_block_starts_bit_exact():
    rng = np.random.default_rng(5)
    for trial in range(40):
        rows = int(rng.integers(1, 3000))
        counts = rng.integers(0, 9, size=rows) * (rng.random(rows) < 0.7)
        rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        nnz = int(rp[-1])
        chunk = int(rng.integers(1, 300))
        nb = -(-nnz // chunk) if nnz else 0
        cols = np.concatenate([np.arange(c) for c in counts]) if nnz else np.zeros(0, np.int64)
        mat = CsrMatrix(rows, 8, rp, cols, np.ones(nnz))
        da = DeviceCsr.from_host(mat)
        got = device_block_starts(da, chunk, nb).cpu().numpy().astype(np.int64)
        assert got.tolist() == compute_block_starts(rp, chunk, nb).tolist()
        assert got.tolist() == oracle.block_starts(rp, chunk, nb).tolist()


def test_accumulate_into_c0():
    a = random_csr(64, 64, 0.2, seed=7)
    b = random_dense(64, 8, seed=8)
    c0 = random_dense(64, 8, seed=9)
    want = oracle.spmm_f64(a.row_ptr, a.col_idx, a.vals, b.vals.reshape(64, 8), 8).reshape(-1) + c0.vals
    for text in ("nnz:32,col:1,r:1", "row:2,col:2,r:1", "row:1/4,col:4,r:4", "nnz:1,col:1,r:8",
                 "nnz:1,col:2,r:1"):
        k = build_kernel(parse_point(text), KernelConfig(8, 256), a)
        got, _ = run(k, a, b, c0=c0)
        np.testing.assert_allclose(got.vals, want, rtol=0, atol=1e-12)
        assert np.array_equal(c0.vals, random_dense(64, 8, seed=9).vals)  # c0 not aliased


def test_empty_matrix_and_empty_rows():
    empty = CsrMatrix(16, 16, np.zeros(17, dtype=np.int64), [], [])
    b = random_dense(16, 4, seed=1)
    for text in ("nnz:1,col:1,r:32", "row:32,col:1,r:1", "nnz:32,col:1,r:1", "row:1/32,col:1,r:32"):
        k = build_kernel(parse_point(text), KernelConfig(4, 256), empty)
        got, m = run(k, empty, b)
        assert not np.any(got.vals)
    c0 = random_dense(16, 4, seed=3)
    k = build_kernel(parse_point("nnz:1,col:1,r:32"), KernelConfig(4, 256), empty)
    got, _ = run(k, empty, b, c0=c0)
    assert np.array_equal(got.vals, c0.vals)


def test_run_errors_mirror_reference():
    a = random_csr(32, 32, 0.2, seed=7)
    b = random_dense(32, 4, seed=8)
    k = build_kernel(parse_point("nnz:32,col:1,r:1"), KernelConfig(4, 256), a)
    with pytest.raises(ValueError):
        run(k, a, b, precision="half")
    with pytest.raises(ValueError):
        run(k, a, random_dense(31, 4, seed=1))
    with pytest.raises(ValueError):
        run(k, a, b, c0=random_dense(31, 4, seed=1))


def test_verify_point_reports():
    a = random_csr(16, 16, 0.25, seed=3)
    cfg = KernelConfig(4, 256)
    rep = verify_point(a, parse_point("nnz:1,col:1,r:32"), cfg)
    assert rep.status == "pass" and rep.family == "nnz-one" and rep.kernel == "spmm_nnz_one"
    assert rep.max_rel_error <= 1e-12
    rep = verify_point(a, parse_point("row:1,col:1/2,r:1"), cfg)
    assert rep.status == "no_template" and rep.max_rel_error is None
    rep = verify_point(a, parse_point("nnz:32,col:1,r:1"), cfg, tolerance=0.0, precision="single")
    assert rep.status == "fail" and rep.max_rel_error > 0


@pytest.mark.parametrize("gsz", [1, 2, 4, 8, 16, 32])
def test_device_group_macros_match_reference(gsz):
    z = np.load(GOLDEN / "group_primitives.npz")
    for kind, fn in (("atomic", exec_atomic_add_group), ("seg", exec_seg_reduce_group)):
        out = np.zeros(512)
        wb = fn(z[f"{kind}|{gsz}|idx"], z[f"{kind}|{gsz}|val"], out, z[f"{kind}|{gsz}|active"],
                group_size=gsz)
        assert wb == int(z[f"{kind}|{gsz}|wb"][0])
        np.testing.assert_allclose(out, z[f"{kind}|{gsz}|out"], rtol=0, atol=1e-9)


def test_device_group_macros_reference_gate_and_faults():
    # test_acceptance.py:152-181 -- 10,016 random groups per width, 80% active
    rng = np.random.default_rng(97)
    for gsz in (2, 4, 8, 16, 32):
        lanes = 10_016 * gsz
        val = rng.uniform(-1, 1, lanes)
        active = rng.random(lanes) < 0.8
        idx = np.repeat(rng.integers(0, 512, 10_016), gsz)
        got, want = np.zeros(512), np.zeros(512)
        assert exec_atomic_add_group(idx, val, got, active, group_size=gsz) == \
            oracle.serial_atomic_add(idx, val, active, want, gsz)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-9)
        idx = np.sort(rng.integers(0, 512, (10_016, gsz)), axis=1).ravel()
        got, want = np.zeros(512), np.zeros(512)
        assert exec_seg_reduce_group(idx, val, got, active, group_size=gsz) == \
            oracle.serial_seg_reduce(idx, val, active, want, gsz)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-9)
    # faults (test_sim.py:94-131)
    with pytest.raises(SimulationFault):
        exec_atomic_add_group(np.array([3, 4, 3, 3]), np.ones(4), np.zeros(8), group_size=4)
    assert exec_atomic_add_group(np.array([3, 4, 3, 3]), np.ones(4), np.zeros(8),
                                 np.array([True, False, True, True]), group_size=4) == 1
    with pytest.raises(SimulationFault) as e:
        exec_seg_reduce_group(np.array([2, 1, 3, 4]), np.ones(4), np.zeros(8), group_size=4)
    assert e.value.lane == 1
    with pytest.raises(ValueError):
        exec_atomic_add_group(np.zeros(5, int), np.zeros(5), np.zeros(4), group_size=4)
    out = np.zeros(8)
    assert exec_seg_reduce_group(np.array([5, 5, 5, 5]), np.ones(4), out, group_size=2) == 2
    assert out[5] == 4.0


@pytest.mark.parametrize("variant", [1, 2, 5])
def test_nnz_multiple_walk_variants(zoo, variant):
    """Both nnz-multiple walks (register-staged, TMA-staged) on the zoo and
    config 1, including g that does not divide the TMA tile evenly."""
    sim = {(r["matrix"], r["n"], r["point"]): r for r in
           json.loads((GOLDEN / "sim_metrics.json").read_text())}
    for n in (4, 8):
        cfg = KernelConfig(n=n, p=256)
        pts = [pt for pt in templated(n, 256) if str(pt).startswith("nnz:") and
               not str(pt).startswith("nnz:1,")]
        assert pts
        for label, mat, b_seed in zoo:
            b = random_dense(mat.num_cols, n, seed=b_seed)
            want = oracle_f32(mat, b, n)
            for pt in pts:
                k = build_kernel(pt, cfg, mat)
                got, m = run(k, mat, b, precision="single", hw_variant=variant)
                assert oracle.max_rel_error(got.vals, want) <= F32_TOL, (label, str(pt))
                assert m.atomic_ops == sim[(label, n, str(pt))]["atomic_ops"]
    a = random_csr(4096, 4096, 0.01, seed=1)
    b = random_dense(4096, 32, seed=2)
    want = oracle_f32(a, b, 32)
    for text, p in (("nnz:32,col:4,r:1", 1024), ("nnz:2,col:4,r:1", 1024), ("nnz:16,col:2,r:1", 1024)):
        k = build_kernel(parse_point(text), KernelConfig(32, p), a)
        got, m = run(k, a, b, precision="single", hw_variant=variant)
        assert oracle.max_rel_error(got.vals, want) <= F32_TOL, text
        st = oracle.block_starts(a.row_ptr, k.chunk, k.grid_size)
        assert m.atomic_ops == oracle.writebacks(k.family, a.row_ptr, 32, k.grid_size, starts=st,
                                                 npb=k.chunk, r=k.r, chunk=k.chunk, g=k.g)


def test_reference_objects_are_accepted():
    """sim.run takes the reference's own LoweredKernel / CsrMatrix / DenseMatrix
    (duck-typed), the zero-code switch of INTEGRATION.md section 1."""
    from types import SimpleNamespace

    a = random_csr(300, 200, 0.05, seed=4)
    b = random_dense(200, 8, seed=5)
    ref_a = SimpleNamespace(num_rows=a.num_rows, num_cols=a.num_cols, row_ptr=a.row_ptr,
                            col_idx=a.col_idx, vals=a.vals, nnz=a.nnz)
    ref_b = SimpleNamespace(num_rows=b.num_rows, num_cols=b.num_cols, vals=b.vals)
    want = oracle.spmm_f64(a.row_ptr, a.col_idx, a.vals, b.vals.reshape(200, 8), 8)
    for text, p in (("nnz:32,col:4,r:1", 1024), ("nnz:1,col:2,r:8", 256), ("row:1/8,col:1,r:8", 256)):
        ours = build_kernel(parse_point(text), KernelConfig(8, p), a)
        ref_k = SimpleNamespace(name=ours.name, body=(), grid_size=ours.grid_size,
                                block_size=ours.block_size, block_starts=ours.block_starts,
                                family=ours.family, point=text)
        got, m = run(ref_k, ref_a, ref_b)
        assert oracle.max_rel_error(got.vals, want) <= F64_TOL
        assert m.grid_size == ours.grid_size


def test_config1_every_candidate_every_walk():
    """Every candidate of the B200 knob grid (g up to 512, every walk variant
    the point admits) on config 1 at N=32, float32, within 1e-5 of the
    float64 reference; the device reference itself is pinned to the CPU
    oracle first (tools/parity_sweep.py runs the same check at configs 2-4)."""
    import torch

    from paper_2209_02882_b200 import _native
    from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, reference_spmm_f64, spmm
    from paper_2209_02882_b200.selector import candidates, plan_for

    dev = torch.device("cuda", 0)
    a_h = random_csr(4096, 4096, 0.01, seed=1)
    b_h = random_dense(4096, 32, seed=2)
    a = DeviceCsr(4096, 4096, torch.as_tensor(np.asarray(a_h.row_ptr, np.int32), device=dev),
                  torch.as_tensor(np.asarray(a_h.col_idx, np.int32), device=dev),
                  torch.as_tensor(np.asarray(a_h.vals, np.float32), device=dev))
    b = torch.as_tensor(np.asarray(b_h.vals, np.float32).reshape(4096, 32), device=dev)
    want = reference_spmm_f64(a, b, 32)
    assert np.array_equal(want.cpu().numpy(), oracle_f32(a_h, b_h, 32).reshape(4096, 32))
    c = torch.empty((4096, 32), dtype=torch.float32, device=dev)
    rp = np.asarray(a_h.row_ptr, np.int64)
    runs = 0
    for cand in candidates(32):
        k = plan_for(cand, 32, 4096, 4096, rp)
        aux = prepare_aux(k, a, row_ptr_host=rp)
        c.fill_(float("nan"))
        try:
            spmm(k, a, b, c, aux=aux, hw_block=cand.hw_block, hw_variant=cand.hw_variant)
        except _native.SgapError as e:
            assert e.status == _native.ERR_ARG  # variant not applicable to this point
            continue
        err = float(((c.double() - want).abs() / (want.abs() + 1)).max())
        assert err <= F32_TOL, (cand.label(), err)
        runs += 1
    assert runs > 250


@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
def test_device_shard_cuts_bit_exact(k):
    """partition.shard_starts_device == partition.shard_starts (the multi-GPU
    cut points) on R-MAT, a matrix with leading/trailing empty
    rows and an empty one."""
    from paper_2209_02882_b200 import generators as G
    from paper_2209_02882_b200.partition import shard_starts, shard_starts_device

    rm = G.rmat(14, 16, seed=2)
    cases = [rm.row_ptr.numpy().astype(np.int64),
             np.array([0, 0, 0, 3, 3, 7, 7, 7, 9, 9, 9], np.int64),
             np.zeros(6, np.int64)]
    for rp in cases:
        got = shard_starts_device(torch.as_tensor(rp.astype(np.int32), device="cuda"), k)
        assert np.array_equal(got.cpu().numpy(), shard_starts(rp, k)), (k, rp[:8])


def test_nnz_one_segment_walk_variant(zoo):
    """nnz-one hw variant 1: every aligned segment group walked serially by
    lanes along the columns (the register walk with g = r) instead of the
    shuffle scan -- identical writeback counts to the reference simulator
    on the zoo (including the padded tail group), both precisions, and on
    config 1 against the oracle's writeback restatement."""
    sim = {(r["matrix"], r["n"], r["point"]): r for r in
           json.loads((GOLDEN / "sim_metrics.json").read_text())}
    golden = np.load(GOLDEN / "zoo_oracle.npz")
    runs = 0
    for n in (4, 8):
        cfg = KernelConfig(n=n, p=256)
        pts = [pt for pt in templated(n, 256) if str(pt).startswith("nnz:1,")]
        assert pts
        for label, mat, b_seed in zoo:
            b = random_dense(mat.num_cols, n, seed=b_seed)
            want32 = oracle_f32(mat, b, n)
            for pt in pts:
                k = build_kernel(pt, cfg, mat)
                got, m = run(k, mat, b, precision="single", hw_variant=1)
                assert oracle.max_rel_error(got.vals, want32) <= F32_TOL, (label, str(pt))
                assert m.atomic_ops == sim[(label, n, str(pt))]["atomic_ops"], (label, n, str(pt))
                got64, m64 = run(k, mat, b, precision="double", hw_variant=1)
                assert oracle.max_rel_error(got64.vals, golden[f"{label}|{n}"]) <= F64_TOL
                assert m64.atomic_ops == m.atomic_ops
                runs += 1
    a = random_csr(4096, 4096, 0.01, seed=1)
    b = random_dense(4096, 32, seed=2)
    want = oracle_f32(a, b, 32)
    for text, p in (("nnz:1,col:4,r:8", 256), ("nnz:1,col:1,r:32", 1024), ("nnz:1,col:2,r:1", 256)):
        k = build_kernel(parse_point(text), KernelConfig(32, p), a)
        got, m = run(k, a, b, precision="single", hw_variant=1)
        assert oracle.max_rel_error(got.vals, want) <= F32_TOL, text
        st = oracle.block_starts(a.row_ptr, k.chunk, k.grid_size)
        assert m.atomic_ops == oracle.writebacks(k.family, a.row_ptr, 32, k.grid_size, starts=st,
                                                 npb=k.chunk, r=k.r), text
    print("nnz-one segment walk:", runs, "zoo runs")
