"""Pin the CPU oracle (oracle/) against fixtures produced by the reference
itself (tests/golden/make_golden.py imports /root/reference/pkg/src).

Every assertion here is exact: the oracle restates integer partition logic and
an f64 accumulation order, so it must reproduce the reference bit for bit."""

import hashlib
import json

import numpy as np
import pytest

import oracle
from paper_2209_02882_b200.lowering import KernelConfig
from paper_2209_02882_b200.matrices import random_csr, random_dense
from paper_2209_02882_b200.runner import build_kernel
from paper_2209_02882_b200.space import parse_point

from conftest import GOLDEN


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def space():
    return json.loads((GOLDEN / "space.json").read_text())


def test_zoo_regenerates_bit_identically(zoo):
    meta = {m["label"]: m for m in json.loads((GOLDEN / "zoo_meta.json").read_text())}
    assert len(meta) == len(zoo) == 20
    for label, mat, b_seed in zoo:
        m = meta[label]
        assert m["b_seed"] == b_seed
        assert sha(mat.row_ptr) == m["row_ptr_sha"], label
        assert sha(mat.col_idx) == m["col_idx_sha"], label
        assert sha(mat.vals) == m["vals_sha"], label


def test_oracle_bit_identical_to_reference_on_zoo(zoo):
    golden = np.load(GOLDEN / "zoo_oracle.npz")
    for label, mat, b_seed in zoo:
        for n in (4, 8):
            b = random_dense(mat.num_cols, n, seed=b_seed)
            got = oracle.spmm_f64(mat.row_ptr, mat.col_idx, mat.vals,
                                  b.vals.reshape(mat.num_cols, n), n)
            want = golden[f"{label}|{n}"]
            assert np.array_equal(got.reshape(-1), want), label


def test_oracle_bit_identical_on_config1():
    cfg = json.loads((GOLDEN / "cfg1.json").read_text())
    a = random_csr(4096, 4096, 0.01, seed=1)
    b = random_dense(4096, 32, seed=2)
    assert a.nnz == cfg["nnz"] == 167772
    assert sha(a.row_ptr) == cfg["row_ptr_sha"]
    assert sha(a.col_idx) == cfg["col_idx_sha"]
    assert sha(a.vals) == cfg["vals_sha"]
    assert sha(b.vals) == cfg["b_sha"]
    got = oracle.spmm_f64(a.row_ptr, a.col_idx, a.vals, b.vals.reshape(4096, 32), 32)
    assert sha(got.reshape(-1)) == cfg["oracle_sha"]
    # the device-layout entry (int32 indices, float32 operands widened) equals
    # the reference oracle run on the float32-rounded operands
    got32 = oracle.spmm_f64(a.row_ptr.astype(np.int32), a.col_idx.astype(np.int32),
                            a.vals.astype(np.float32), b.vals.astype(np.float32).reshape(4096, 32), 32)
    assert sha(got32.reshape(-1)) == cfg["oracle_f32in_sha"]
    # thread count never changes a bit
    one = oracle.spmm_f64(a.row_ptr, a.col_idx, a.vals, b.vals.reshape(4096, 32), 32, threads=1)
    assert np.array_equal(one, got)


def test_block_starts_and_search_known_cases(space):
    for case in space["starts_cases"]:
        rp = np.asarray(case["row_ptr"], np.int64)
        got = oracle.block_starts(rp, case["chunk"], case["num_blocks"])
        assert got.tolist() == case["starts"]
        assert oracle.brute_block_starts(rp, case["chunk"], case["num_blocks"]) == case["starts"]
        assert oracle.search_before(rp, case["lo"], case["hi"], case["target"]) == case["search"]


def test_reference_known_answers():
    # lowering.compute_block_starts / binary_search_before known answers
    # (pkg/tests/test_lowering.py:48-84)
    assert oracle.block_starts(np.array([0, 2, 5, 5, 9]), 4, 3).tolist() == [0, 1, 3, 4]
    a = [0, 2, 5, 5, 9]
    assert [oracle.search_before(a, 0, 5, t) for t in (0, 4, 5, 100, -1)] == [0, 1, 3, 4, 0]
    assert oracle.search_before(a, 2, 4, 100) == 3


def _starts_for(k, mat):
    return oracle.block_starts(mat.row_ptr, k.chunk, k.grid_size)


def test_writeback_counts_match_reference_simulator(zoo):
    """SimMetrics.atomic_ops of sim.run for every templated point on the zoo
    (2640 reference simulations) restated by the C oracle."""
    rows = json.loads((GOLDEN / "sim_metrics.json").read_text())
    mats = {label: mat for label, mat, _ in zoo}
    assert len(rows) == 2640
    for r in rows:
        mat = mats[r["matrix"]]
        k = build_kernel(parse_point(r["point"]), KernelConfig(r["n"], r["p"]), mat)
        assert (k.grid_size, k.block_size, k.family) == (r["grid"], r["block"], r["family"])
        st = _starts_for(k, mat) if k.family.startswith("nnz") else None
        got = oracle.writebacks(k.family, mat.row_ptr, r["n"], k.grid_size, starts=st,
                                npb=k.chunk, r=k.r, chunk=k.chunk, g=k.g)
        assert got == r["atomic_ops"], r


def test_writeback_counts_config1_simulator_pins():
    cfg = json.loads((GOLDEN / "cfg1.json").read_text())
    if not cfg["sim"]:
        pytest.skip("cfg1 simulator pins not generated")
    a = random_csr(4096, 4096, 0.01, seed=1)
    for s in cfg["sim"]:
        k = build_kernel(parse_point(s["point"]), KernelConfig(32, s["p"]), a)
        assert (k.grid_size, k.block_size) == (s["grid"], s["block"])
        st = _starts_for(k, a) if k.family.startswith("nnz") else None
        got = oracle.writebacks(k.family, a.row_ptr, 32, k.grid_size, starts=st, npb=k.chunk,
                                r=k.r, chunk=k.chunk, g=k.g)
        assert got == s["atomic_ops"], s


@pytest.mark.parametrize("gsz", [1, 2, 4, 8, 16, 32])
def test_serial_group_restatements_match_reference(gsz):
    z = np.load(GOLDEN / "group_primitives.npz")
    for kind, fn in (("atomic", oracle.serial_atomic_add), ("seg", oracle.serial_seg_reduce)):
        out = np.zeros(512)
        wb = fn(z[f"{kind}|{gsz}|idx"], z[f"{kind}|{gsz}|val"], z[f"{kind}|{gsz}|active"], out, gsz)
        assert wb == int(z[f"{kind}|{gsz}|wb"][0])
        np.testing.assert_allclose(out, z[f"{kind}|{gsz}|out"], rtol=0, atol=1e-12)


def test_spec_known_answers_for_group_macros():
    # SPEC.md:386-396 and pkg/tests/test_sim.py:140-147
    out = np.zeros(8)
    assert oracle.serial_seg_reduce([5, 5, 7, 7], [1, 2, 3, 4], [1] * 4, out, 4) == 2
    assert out[5] == 3 and out[7] == 7
    out = np.zeros(8)
    assert oracle.serial_atomic_add([3, 3, 3, 3], [1, 2, 3, 4], [1] * 4, out, 4) == 1
    assert out[3] == 10
    out = np.zeros(8)
    assert oracle.serial_seg_reduce([5, 5, 5, 5], [1.0] * 4, [1] * 4, out, 2) == 2
    assert out[5] == 4.0
