"""The C ABI boundary: libsgap.so loads without a GPU, exports exactly what
include/sgap.h declares, and host-only entry points validate arguments.
No compute call is made here (no GPU in the CPU suite)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2209_02882_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "sgap.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char \*)\s*(sgap_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(sgap_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    L = _native.lib()
    for name in declared_symbols():
        assert hasattr(L, name)


def test_abi_version_and_status_strings():
    L = _native.lib()
    assert L.sgap_abi_version() == 5
    assert _native.status_string(_native.ERR_NO_TEMPLATE) == "no template covers the point"
    assert _native.status_string(99) == "unknown status"


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_argument_validation_without_device():
    L = _native.lib()
    k = _native.Kernel()
    assert L.sgap_run(None, None, None, None, 0, None, None) == _native.ERR_ARG
    assert L.sgap_long_row_threshold(None, 0) == -1
    k.n, k.c = 4, 1
    a = _native.Csr()
    # sgap_run takes only a plan built by sgap_plan (ABI v4+): a zeroed struct is rejected
    plan = _native.Plan()
    assert L.sgap_run(ctypes.byref(plan), ctypes.byref(a), None, None, 0, None, None) == _native.ERR_ARG
    # the planner: workspace sizing is host-only; bad dtype / config / shape are caught first
    nb = ctypes.c_size_t(0)
    assert L.sgap_plan_workspace_bytes(ctypes.byref(k), ctypes.byref(a), 7, 0,
                                       ctypes.byref(nb)) == _native.ERR_PRECISION
    k.family, k.g, k.chunk, k.grid_size = _native.FAMILY_IDS["nnz-multiple"], 256, 256, 4
    a.num_rows, a.num_cols, a.nnz = 100, 100, 1000
    assert L.sgap_plan_workspace_bytes(ctypes.byref(k), ctypes.byref(a), 0, 0,
                                       ctypes.byref(nb)) == _native.OK
    # block starts + row ids + stats at least; float32 adds the long-row table
    assert nb.value >= 4 * 5 + 4 * 1000
    nb64 = ctypes.c_size_t(0)
    assert L.sgap_plan_workspace_bytes(ctypes.byref(k), ctypes.byref(a), 1, 0,
                                       ctypes.byref(nb64)) == _native.OK
    assert nb64.value < nb.value  # float64 values: no table
    a.nnz = -1
    assert L.sgap_plan_workspace_bytes(ctypes.byref(k), ctypes.byref(a), 0, 0,
                                       ctypes.byref(nb)) == _native.ERR_SHAPE
    a.nnz = 1000
    assert L.sgap_plan(ctypes.byref(k), ctypes.byref(a), 0, 0, None, 0, ctypes.byref(plan),
                       None) == _native.ERR_ARG  # no row_ptr / workspace
    k.n, k.c = 6, 4
    assert L.sgap_plan_workspace_bytes(ctypes.byref(k), ctypes.byref(a), 0, 0,
                                       ctypes.byref(nb)) == _native.ERR_CONFIG
    assert L.sgap_validate_csr(None, None, None, None) == _native.ERR_ARG
    assert L.sgap_block_starts(None, 4, 0, 1, None, None) == _native.ERR_ARG
    assert L.sgap_seg_reduce_group(None, None, None, 5, 4, None, 0, 0, None, None, None) == _native.ERR_ARG
    assert L.sgap_atomic_add_group(None, None, None, 8, 3, None, 0, 0, None, None, None) == _native.ERR_ARG
    # Matrix Market ingest entry points
    assert L.sgap_mm_line_flags(None, -1, None, None, None) == _native.ERR_ARG
    assert L.sgap_mm_line_flags(None, 0, None, None, None) == _native.OK
    assert L.sgap_mm_parse(None, 10, None, 1, 2**31, 4, None, None, None, None, None, None,
                           None) == _native.ERR_SHAPE
    assert L.sgap_mm_parse(None, 10, None, 1, 4, 4, None, None, None, None, None, None,
                           None) == _native.ERR_ARG
    assert L.sgap_mm_expand(-1, None, None, None, None, None, 0, None, None, None) == _native.ERR_ARG
    assert L.sgap_mm_sum_runs(0, None, None, None, 0, None, None, None, None) == _native.OK


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_PATH", tmp_path / "nope.so")
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(_native.NativeLibraryError):
        _native.lib()


def test_ctypes_structs_match_the_c_header(tmp_path):
    """Every ctypes mirror in _native.py has the C header's size and field
    offsets (gcc on include/sgap.h), so a field added to one side only
    (ABI v5 added d_panel_b / panel_lanes to sgap_aux_t) fails here, not as
    a misread plan on the GPU."""
    import shutil
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    mirrors = {"sgap_point_t": _native.Point, "sgap_kernel_t": _native.Kernel,
               "sgap_csr_t": _native.Csr, "sgap_aux_t": _native.Aux, "sgap_plan_t": _native.Plan}
    # ctypes names the two elements of the C arrays d_union_off[2] / d_union[2]
    alias = {"d_union_off4": "d_union_off[0]", "d_union_off8": "d_union_off[1]",
             "d_union4": "d_union[0]", "d_union8": "d_union[1]"}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sgap.h"', "int main(void) {"]
    for cname, py in mirrors.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            member = alias.get(fname, fname) if cname == "sgap_aux_t" else fname
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {member}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(ROOT / "include"), str(src), "-o", str(exe)],
                   check=True, capture_output=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n"):
        if line:
            cname, field, value = line.split()
            got[cname, field] = int(value)
    for cname, py in mirrors.items():
        assert got[cname, "size"] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[cname, fname] == getattr(py, fname).offset, (cname, fname)
