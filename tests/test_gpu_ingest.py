"""Device Matrix Market ingest (paper_2209_02882_b200.ingest) against the host
parser (matrices.loads_matrix_market, pinned to the reference's cases in
test_matrices.py): identical row_ptr / col_idx / bit-identical values, and
identical errors (message and line number)."""

import numpy as np
import pytest
import torch

from paper_2209_02882_b200.ingest import load_matrix_market_device
from paper_2209_02882_b200.matrices import MatrixFormatError, loads_matrix_market, random_csr

pytestmark = pytest.mark.gpu


def same(text):
    want = loads_matrix_market(text)
    got = load_matrix_market_device(text)
    assert (got.num_rows, got.num_cols) == (want.num_rows, want.num_cols)
    assert np.array_equal(got.row_ptr.cpu().numpy(), want.row_ptr)
    assert np.array_equal(got.col_idx.cpu().numpy(), want.col_idx)
    gv, wv = got.vals.cpu().numpy(), np.asarray(want.vals, np.float64)
    nan = np.isnan(wv)  # NaN payloads differ between x86 and the GPU; positions must not
    assert np.array_equal(np.isnan(gv), nan)
    assert np.array_equal(gv[~nan].view(np.int64), wv[~nan].view(np.int64))
    return got


def test_reference_cases():
    same("""%%MatrixMarket matrix coordinate real general
% a comment line
3 4 3
1 1 2.5
3 4 -1.0
2 2 7
""")
    same("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 4\n2 1 5\n")
    same("%%MatrixMarket matrix coordinate real general\n1 1 2\n1 1 1.5\n1 1 2.5\n")
    same("%%MatrixMarket matrix coordinate real general\n3 3 0\n")
    same("%%MatrixMarket matrix coordinate real general\n3 3 1\n\n% c\n2 3 1e-3")


def _mm(rng, rows, cols, n, sym, fmt, dup_heavy=False):
    r = rng.integers(1, rows + 1, n)
    c = rng.integers(1, cols + 1, n)
    if dup_heavy:  # long runs of the same coordinate: numpy's pairwise order matters
        r[: n // 2] = 1
        c[: n // 2] = 1
    if sym:
        r, c = np.maximum(r, c), np.minimum(r, c)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-12, 12, n)
    lines = []
    for i in range(n):
        if rng.random() < 0.02:
            lines.append("% comment " + str(i))
        if rng.random() < 0.01:
            lines.append("   ")
        lines.append(f"{r[i]} \t{c[i]}  {fmt(v[i], rng)}")
    kind = "symmetric" if sym else "general"
    return f"%%MatrixMarket matrix coordinate real {kind}\n% gen\n{rows} {cols} {n}\n" + "\n".join(lines) + "\n"


FORMATS = [
    lambda x, rng: repr(float(x)),                 # 17-digit repr: Eisel-Lemire on the device
    lambda x, rng: f"{x:.6e}",                     # fast path
    lambda x, rng: f"{x:.3f}",
    lambda x, rng: ["1_0.5", "inf", "-Infinity", "nan", "1e400", "4.9e-324", "+.5", "5.", "-0",
                    "0.1000000000000000055511151231257827", repr(float(x))][rng.integers(0, 11)],
]


@pytest.mark.parametrize("sym", [False, True])
@pytest.mark.parametrize("fi", range(len(FORMATS)))
def test_random_texts(sym, fi):
    rng = np.random.default_rng(100 + fi + 10 * sym)
    same(_mm(rng, 300, 300 if sym else 200, 4000, sym, FORMATS[fi]))


def test_duplicate_runs_sum_in_numpy_order():
    rng = np.random.default_rng(5)
    for n in (9, 17, 200, 1000):
        same(_mm(rng, 4, 4, n, False, FORMATS[0], dup_heavy=True))


def _hard_decimals(rng, n):
    """Decimal strings across the binary64 range that Clinger's fast path
    cannot take: 17-digit round-trip reprs of random bit patterns, 16-19
    digit mantissas with large exponents, exact halfway cases (2^53 + 1 and
    its neighbours), subnormals and overflow (host), > 19 digits (host)."""
    bits = rng.integers(0, 2**63 - 1, n, dtype=np.int64) & ~np.int64(0x7FF0000000000000) | \
        (rng.integers(1, 2046, n, dtype=np.int64) << 52)
    out = [repr(float(x)) for x in bits.view(np.float64)]
    out += [f"{int(m)}e{int(e)}" for m, e in zip(rng.integers(10**15, 10**18, n),
                                                  rng.integers(-340, 290, n))]
    out += [f"{x:.16e}" for x in rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)]
    out += ["9007199254740993", "9007199254740995", "9007199254740992.5", "18014398509481986",
            "2.2250738585072014e-308", "1.7976931348623157e308", "4.9e-324", "2.5e-320", "1e309",
            "8.98846567431158e307", "7.2057594037927933e16", "1e23", "0.1", "-1.5e-300",
            "1.00000000000000011102230246251565404236316680908203125", "9999999999999999999",
            "12345678901234567890e-10"]
    return out


def test_correctly_rounded_decimals_on_device():
    """Every value bit-identical to float(); normal finite results of <= 19
    significant digits are converted on the device (Eisel-Lemire), only
    subnormal / overflowing / > 19-digit tokens reach the host."""
    rng = np.random.default_rng(17)
    vals = _hard_decimals(rng, 4000)
    n = len(vals)
    text = f"%%MatrixMarket matrix coordinate real general\n{n} 1 {n}\n" + \
        "\n".join(f"{i + 1} 1 {v}" for i, v in enumerate(vals)) + "\n"
    stats = {}
    got = load_matrix_market_device(text, stats=stats)
    want = np.array([float(v) for v in vals])
    gv = got.vals.cpu().numpy()
    assert np.array_equal(got.row_ptr.cpu().numpy(), np.arange(n + 1))
    assert np.array_equal(gv.view(np.int64), want.view(np.int64))
    host = sum(1 for v in vals if len(v.lstrip("-").split("e")[0].replace(".", "").lstrip("0")) > 19
               or not (2.2250738585072014e-308 <= abs(float(v)) < float("inf")))
    assert stats["lines"] == n
    assert stats["host_floats"] + stats["host_lines"] <= host, (stats, host)


def test_shapes_beyond_32_bit_keys_stay_exact():
    # (row << 32 | col) keys need 31-bit shapes; larger ones take the host parser
    same("%%MatrixMarket matrix coordinate real general\n5 4294967300 3\n"
         "1 4294967299 1.5\n1 2 2.5\n5 4294967300 -1\n")


def test_crlf_and_header_comments():
    text = "%%MatrixMarket matrix coordinate real general\r\n%c\r\n\r\n2 2 2\r\n1 1 0.5\r\n2 2 -3\r\n"
    same(text)
    same(text.replace("\r\n", "\n").replace("0.5\n", "0.5\r\r\n"))  # lone \r: host path


@pytest.mark.parametrize("text", [
    "",
    "%%MatrixMarket matrix coordinate real general\n",
    "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0 4\n2 2 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2 abc\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n% c\n\n0 2 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1e\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 2\n9 9 x\n",  # non-numeric wins over range
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 2\n1 1 3\n\n",
])
def test_errors_match_host(text):
    with pytest.raises(MatrixFormatError) as want:
        loads_matrix_market(text)
    with pytest.raises(MatrixFormatError) as got:
        load_matrix_market_device(text)
    assert (str(got.value), got.value.line) == (str(want.value), want.value.line)


def test_large_matrix_round_trip_and_spmm_layout():
    a = random_csr(3000, 2000, 0.01, seed=4)
    rows = np.repeat(np.arange(a.num_rows), np.diff(a.row_ptr))
    body = "\n".join(f"{r + 1} {c + 1} {float(v)!r}" for r, c, v in zip(rows, a.col_idx, a.vals))
    text = f"%%MatrixMarket matrix coordinate real general\n3000 2000 {a.nnz}\n{body}\n"
    got = same(text)
    d = got.to_csr(torch.float32)
    assert d.row_ptr.dtype == torch.int32 and d.vals.dtype == torch.float32
    assert np.array_equal(d.row_ptr.cpu().numpy(), a.row_ptr)
