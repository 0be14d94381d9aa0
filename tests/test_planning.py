"""Host planning (point grammar, legality, template gates, launch geometry,
block starts) against the reference's own outputs (tests/golden/space.json),
for both the Python mirror and the C planner in libsgap.so."""

import ctypes
import hashlib
import itertools
import json

import numpy as np
import pytest
from fractions import Fraction

from paper_2209_02882_b200 import _native
from paper_2209_02882_b200.lowering import (KernelConfig, LoweringError, binary_search_before,
                                            compute_block_starts)
from paper_2209_02882_b200.matrices import CsrMatrix, random_csr
from paper_2209_02882_b200.runner import build_kernel, enumerate_report
from paper_2209_02882_b200.space import (AmountKind, DataKind, PointError, da_spmm_points,
                                         enumerate_fine_grained, enumerate_space, legality_rule,
                                         parse_point)
from paper_2209_02882_b200.templates import IllegalPointError, algorithm_template, template_family

from conftest import GOLDEN

GEOM = {
    "emit64": lambda: random_csr(64, 64, 0.0625, seed=1),
    "dense96": lambda: random_csr(96, 96, 0.5, seed=3),
    "tall300": lambda: random_csr(300, 16, 0.1, seed=4),
    "empty16": lambda: CsrMatrix(16, 16, np.zeros(17, dtype=np.int64), [], []),
    "lead_empty": lambda: CsrMatrix(6, 4, [0, 0, 0, 2, 2, 5, 5], [0, 3, 0, 1, 2], [1.0] * 5),
}


@pytest.fixture(scope="module")
def space():
    return json.loads((GOLDEN / "space.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def test_enumeration_matches_reference(space):
    enum = enumerate_space()
    assert [str(p) for p in enum.legal] == space["legal"]
    assert {str(p): r for p, r in enum.rejected} == space["rejected"]
    assert len(enum.legal) == 333 and len(enum.rejected) == 327
    assert [str(p) for p in da_spmm_points()] == space["da_spmm"]


def test_templated_sets_and_geometry_match_reference(space):
    mats = {k: f() for k, f in GEOM.items()}
    for key, entry in space["configs"].items():
        n, p = map(int, key.split(","))
        cfg = KernelConfig(n=n, p=p)
        rep = enumerate_report(cfg)
        assert [e["point"] for e in rep["legal"] if e["templated"]] == entry["templated"], key
        assert {e["point"]: e["family"] for e in rep["legal"]} == entry["families"], key
        for ptxt, per in entry["kernels"].items():
            for mname, want in per.items():
                k = build_kernel(parse_point(ptxt), cfg, mats[mname])
                assert (k.grid_size, k.block_size, k.name, k.family) == \
                    (want["grid"], want["block"], want["name"], want["family"]), (key, ptxt, mname)
                assert (k.block_starts is not None) == ("starts_sha" in want)
                if k.block_starts is not None:
                    assert len(k.block_starts) == want["starts_len"]
                    assert sha(k.block_starts) == want["starts_sha"]
                    if "starts" in want:
                        assert k.block_starts.tolist() == want["starts"]


def _c_point(pt):
    kinds = {AmountKind.RECIPROCAL: 0, AmountKind.ONE: 1, AmountKind.MULTIPLE: 2}
    return _native.Point(0 if pt.data_kind is DataKind.NNZ else 1, kinds[pt.data_amount.kind],
                         pt.data_amount.param or 0, kinds[pt.col_amount.kind],
                         pt.col_amount.param or 0, pt.r)


def test_c_planner_matches_reference(space):
    """sgap_build_kernel (the C ABI planner) against the reference geometry."""
    L = _native.lib()
    mats = {k: f() for k, f in GEOM.items()}
    enum = enumerate_space()
    for pt, rule in enum.rejected:
        assert L.sgap_legality_rule(ctypes.byref(_c_point(pt))) == rule
    for key, entry in space["configs"].items():
        n, p = map(int, key.split(","))
        templated = set(entry["templated"])
        for pt in enum.legal:
            assert L.sgap_legality_rule(ctypes.byref(_c_point(pt))) == 0
            for mname, mat in mats.items():
                out = _native.Kernel()
                rule = ctypes.c_int32(-1)
                st = L.sgap_build_kernel(ctypes.byref(_c_point(pt)), n, p, mat.num_rows, mat.nnz,
                                         ctypes.byref(out), ctypes.byref(rule))
                if str(pt) not in templated:
                    assert st == _native.ERR_NO_TEMPLATE, (key, str(pt))
                    continue
                assert st == _native.OK
                want = entry["kernels"][str(pt)][mname]
                assert (out.grid_size, out.block_size) == (want["grid"], want["block"])
                assert _native.FAMILY_NAMES[out.family] == want["family"]
                assert bool(out.has_block_starts) == ("starts_sha" in want)
                if out.has_block_starts:
                    assert out.grid_size + 1 == want["starts_len"]
        for pt, rule in enum.rejected:
            out = _native.Kernel()
            r = ctypes.c_int32(0)
            st = L.sgap_build_kernel(ctypes.byref(_c_point(pt)), n, p, 4, 4, ctypes.byref(out),
                                     ctypes.byref(r))
            assert st == _native.ERR_ILLEGAL_POINT and r.value == rule


def test_c_planner_rejects_bad_config():
    L = _native.lib()
    pt = _c_point(parse_point("nnz:1,col:1,r:32"))
    out = _native.Kernel()
    for n, p in ((0, 256), (4, 16), (4, 100)):
        assert L.sgap_build_kernel(ctypes.byref(pt), n, p, 4, 4, ctypes.byref(out), None) == _native.ERR_CONFIG


def test_illegal_points_raise_with_rule():
    with pytest.raises(IllegalPointError) as e:
        build_kernel(parse_point("nnz:1/2,col:1,r:1"), KernelConfig(4, 256), random_csr(8, 8, 0.5, 1))
    assert e.value.rule == 1
    with pytest.raises(IllegalPointError) as e:
        template_family(parse_point("row:1/8,col:1,r:4"))
    assert e.value.rule == 2
    with pytest.raises(IllegalPointError) as e:
        template_family(parse_point("row:1/8,col:1/2,r:8"))
    assert e.value.rule == 3
    assert build_kernel(parse_point("row:1,col:1/2,r:1"), KernelConfig(4, 256),
                        random_csr(8, 8, 0.5, 1)) is None


@pytest.mark.parametrize("text", ["nnz:1,col:4", "nnz:1,col:4,r:x", "foo:1,col:1,r:1",
                                  "nnz:1/1,col:1,r:1", "nnz:1,col:1,r:0", "nnz:a,col:1,r:1",
                                  "nnz:1;col:1;r:1"])
def test_point_syntax_errors(text):
    with pytest.raises(PointError):
        parse_point(text)


def test_point_roundtrip():
    for pt in enumerate_space().legal:
        assert parse_point(str(pt)) == pt
    assert str(parse_point(" nnz : 1 , col : 4 , r : 32 ")) == "nnz:1,col:4,r:32"


def test_kernel_config_validation():
    KernelConfig(1, 32)
    for n, p in ((0, 256), (4, 16), (4, 100)):
        with pytest.raises(ValueError):
            KernelConfig(n, p)


def test_fine_grained_grid_sizes():
    # 90/165/300/375 cells at N = 4/16/64/128
    assert [len(enumerate_fine_grained(n)) for n in (4, 16, 64, 128)] == [90, 165, 300, 375]
    cells = enumerate_fine_grained(6)
    assert all(c.coarsen_size == 2 for c in cells)
    assert cells[0].worker_scale == Fraction(1, 4)
    with pytest.raises(ValueError):
        enumerate_fine_grained(0)


def test_host_block_starts_and_search(space):
    for case in space["starts_cases"]:
        rp = np.asarray(case["row_ptr"], np.int64)
        assert compute_block_starts(rp, case["chunk"], case["num_blocks"]).tolist() == case["starts"]
        assert binary_search_before(rp, case["lo"], case["hi"], case["target"]) == case["search"]
    with pytest.raises(LoweringError):
        compute_block_starts([0, 1], 0, 1)


def test_every_templated_point_has_a_device_kernel():
    """The device dispatch covers every family/c/r/g combination the gates admit."""
    for n, p in itertools.product((1, 2, 4, 8, 16, 32, 64, 128, 256, 512), (32, 256, 1024)):
        for pt in enumerate_space().legal:
            tpl = algorithm_template(pt, KernelConfig(n, p))
            if tpl is None:
                continue
            assert tpl.c in (1, 2, 4)
            if tpl.family == "nnz-one":
                assert tpl.r in (1, 2, 4, 8, 16, 32)
            if tpl.family == "row-reciprocal":
                assert tpl.g in (2, 4, 8, 16, 32)
