"""Host-side pieces of bench.py (no GPU): the roofline formula of SURVEY
8(d), the peak sources, the defaults the driver relies on, and the
reference arm's CPU sampler (the reference's own dense_spmm_oracle from
baseline/_ref on remapped row slices, checked against the oracle)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import oracle  # noqa: E402
from paper_2209_02882_b200.matrices import random_csr  # noqa: E402


def test_defaults_are_the_headline_config():
    args = bench.parse_args([])
    assert args.config == 5 and args.gpus == 1 and args.warmup >= 3
    assert bench.default_n(5) == 128


def test_roofline_picks_the_binding_bound():
    peaks = {"hbm_gbs": 6500.0, "fp32_tflops": 75.0, "hbm_source": "x", "fp32_source": "y"}
    # config 5-like: HBM binds
    r = bench.roofline(16_777_216, 263_430_042, 128, 7_380_480, 16.0, peaks)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    want_bytes = 4 * (16_777_216 + 1) + 8 * 263_430_042 + 4 * 128 * 7_380_480 + 4 * 16_777_216 * 128
    assert r["algorithmic_bytes"] == want_bytes
    assert r["frac"] == pytest.approx(want_bytes / 6500e9 / 16e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    # config 3 at N=256-like: the FP32 FMA term binds
    r3 = bench.roofline(232_965, 114_600_000, 256, 232_965, 10.9, peaks)
    assert r3["bound"] == "fp32_fma" and r3["unit"] == "TFLOP/s"
    assert r3["frac"] == pytest.approx(2 * 114_600_000 * 256 / 75e12 / 10.9e-3)


def test_measured_peaks_has_both_denominators():
    p = bench.measured_peaks()
    assert p["hbm_gbs"] > 1000 and p["fp32_tflops"] > 10
    assert "nominal" in p["fp32_source"]


def test_reference_arm_sampler_matches_the_oracle():
    if bench._ref_import() is None:
        pytest.skip("reference install baseline/_ref absent")
    a = random_csr(300, 500, 0.05, seed=3)
    rp = a.row_ptr.astype(np.int64)
    ci = a.col_idx.astype(np.int32)
    vals = a.vals.astype(np.float32)
    b = np.random.default_rng(1).uniform(-1, 1, (500, 16)).astype(np.float32)
    # one slice through the worker code, in-process: the column remap keeps
    # every product and its order, so the result is bit-identical
    lo, hi = 40, 170
    p0, p1 = int(rp[lo]), int(rp[hi])
    bench._ref_worker_init(rp[lo:hi + 1] - p0, ci[p0:p1], vals[p0:p1], b, 16)
    got = bench._W["oracle"](bench._W["a"], bench._W["b"]).vals.reshape(hi - lo, 16)
    want = oracle.spmm_f64((rp[lo:hi + 1] - p0).astype(np.int32), ci[p0:p1], vals[p0:p1], b, 16)
    assert np.array_equal(got, want)
    value, dt, sample, used = bench.reference_cpu(rp, ci, vals, b, 16, workers=2,
                                                  nnz_per_worker=2000, steps=1, warmup=0)
    assert value > 0 and dt > 0 and used == 2 and "dense_spmm_oracle" in sample
