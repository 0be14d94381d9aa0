"""Selector: the closed-form heuristic's picks for the BASELINE matrix
classes (its regret against the exhaustive device sweep is measured by
tools/selector_regret.py, profiles/r01_selector_regret.json) and the
candidate grid."""

from paper_2209_02882_b200.lowering import KernelConfig
from paper_2209_02882_b200.selector import MatrixStats, candidates, heuristic
from paper_2209_02882_b200.space import parse_point
from paper_2209_02882_b200.templates import algorithm_template

RMAT20 = MatrixStats(1048576, 1048576, 16086639, 15.34, 9.16, 39633, 0.478)
STENCIL160 = MatrixStats(4096000, 4096000, 109215352, 26.66, 0.04, 27, 0.0)
UNIFORM1 = MatrixStats(4096, 4096, 167772, 40.96, 0.15, 66, 0.0)


def test_heuristic_picks_are_templated():
    for st in (RMAT20, STENCIL160, UNIFORM1):
        for n in (1, 2, 3, 4, 8, 16, 32, 64, 128, 256, 512):
            cand = heuristic(st, n)
            assert algorithm_template(parse_point(cand.point), KernelConfig(n=n, p=cand.p)) is not None


RMAT24 = MatrixStats(16777216, 16777216, 263430042, 15.70, 15.59, 238921, 0.56)
CHUNGLU = MatrixStats(232965, 232965, 114492479, 491.5, 3.0, 76000, 0.0)


def test_heuristic_matrix_classes():
    assert heuristic(RMAT20, 128).point.startswith("nnz:")      # power law -> EB walk
    # register-walk flavour: row ids (config 2: short rows, many empty),
    # row_ptr + cold-column hints (config 5: B >> L2), row_ptr (config 3)
    assert heuristic(RMAT20, 128).hw_variant == 5
    assert heuristic(RMAT20, 8).hw_variant == 5
    assert heuristic(RMAT24, 128).hw_variant == 9
    assert heuristic(CHUNGLU, 64).hw_variant == 1
    # B = 238 MB > L2 but a 64-column panel (60 MB) fits half of it: column panels
    assert heuristic(CHUNGLU, 256).hw_variant == 10
    assert heuristic(STENCIL160, 128).point.startswith("row:8")  # regular -> RB
    assert heuristic(STENCIL160, 128).hw_variant == 8             # shifted 4-row blocks
    # and per 128-column panel at N = 256 / 512
    assert (heuristic(STENCIL160, 512).point, heuristic(STENCIL160, 512).hw_variant) == \
        ("row:8,col:4,r:1", 8)
    assert heuristic(STENCIL160, 256).hw_variant == 8
    # 2 / 4 / 8 rows per warp at N = 64 / 32 / 16
    assert heuristic(STENCIL160, 16).hw_variant == 4
    assert {heuristic(STENCIL160, n).hw_variant for n in (32, 64)} == {8}  # shifted, lane groups
    assert heuristic(STENCIL160, 16).point.startswith("row:4")
    assert heuristic(STENCIL160, 4).point == "row:1,col:4,r:1"
    # narrow B on power-law rows: serial segment groups; N=8: short chunks
    assert (heuristic(RMAT20, 4).point, heuristic(RMAT20, 4).hw_variant) == ("nnz:1,col:1,r:16", 1)
    assert heuristic(RMAT20, 8).point.startswith("nnz:64,")
    assert heuristic(UNIFORM1, 4).point == "row:1/8,col:1,r:8"    # flexible group beats r=32
    assert heuristic(UNIFORM1, 32).point == "row:1/2,col:2,r:2"


def test_heuristic_float64_uses_16_byte_vectors():
    # float64 (the reference's default precision): col:2 = one 16-byte vector
    assert ",col:2," in heuristic(RMAT20, 128, esz=8).point
    assert heuristic(STENCIL160, 128, esz=8).point == "row:8,col:2,r:1"
    assert heuristic(STENCIL160, 128, esz=8).hw_variant == 8  # 2 panels of 64 columns


def test_candidate_grid_covers_families_and_walks():
    cands = candidates(128)
    fams = {algorithm_template(parse_point(c.point), KernelConfig(128, c.p)).family for c in cands}
    assert fams == {"nnz-one", "nnz-multiple", "row-multiple", "row-reciprocal"}
    assert any(c.point.startswith("nnz:512") for c in cands)
    # register walks (row_ptr / row ids) and TMA everywhere, lane-staged where N/c >= 32
    # (+ column panels, variant 10, where N/c > 8)
    assert {c.hw_variant for c in cands if c.point.startswith("nnz:64,col:4")} == {1, 5, 9, 2, 3, 10}
    assert {c.hw_variant for c in candidates(32) if c.point.startswith("nnz:64,col:4")} == {1, 5, 9, 2}
    # row-multiple: logical / interleaved, plus a warp per row where N/c == 32
    # (one pass per 32c-column panel where N/c is a larger multiple of 32)
    assert {c.hw_variant for c in cands if c.point.startswith("row:4,col:4")} == {0, 2, 4, 6, 7, 8}
    assert {c.hw_variant for c in cands if c.point.startswith("row:4,col:2")} == {0, 2, 4, 8}
    assert {c.hw_variant for c in candidates(192, p_values=(192,))
            if c.point.startswith("row:4,col:4")} == {0, 2}  # N/c = 48
