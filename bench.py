#!/usr/bin/env python
"""Benchmark: CSR SpMM GFLOP/s (2*nnz*N/t) and HBM GB/s vs roofline on B200.

    python bench.py [--gpus N --steps K --warmup W] [--config 5] [--point P --p 256]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...
    python bench.py --impl reference ...   # the reference's own CPU path

Workload (BASELINE.json configs): the headline is config 5 --
R-MAT scale 24, edge factor 16, Graph500 (0.57,0.19,0.19,0.05), seeded
vertex permutation, duplicates summed, N = 128 dense columns, fp32 -- the
configuration BASELINE's metric is quoted on at 1/2/4/8 B200.  At N GPUs the
same matrix is cut into N nnz-balanced row shards (B replicated, C
row-disjoint, no data-path collective): strong scaling.  ``--config 1..4``
select the other BASELINE shapes (config 2: R-MAT scale 20; ``--weak``
grows it with the world size instead).  ``--gpus N`` without torchrun
re-launches itself under torch.distributed.run with N ranks.

One step = one full SpMM over the resident operands: the zero-fill the
schedule needs + the sm_100a kernel(s) + the long-row fold.  A+B+C exceed the
126 MB L2 (config 5: 19 GB), so no flush is needed between steps.  ``value``
is total GFLOP/s over all ranks with the max-over-ranks device time; ``e2e``
repeats the step through host buffers (pinned H2D of A and B, kernel, D2H of
C inside the timed region) via ``pipeline.HostSpmm``, plus one cold start
(upload, device planning, SpMM, download).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpMM GFLOP/s (2*nnz*N/t)"
UNIT = "GFLOP/s"
FALLBACK_HBM_GBS = 6650.0
SMS = 148
FP32_LANES_PER_SM = 128


# --------------------------------------------------------------------------- setup

def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--weak", action="store_true",
                    help="config 2 only: R-MAT scale 20+log2(world) (weak scaling)")
    ap.add_argument("--n", type=int, default=0, help="dense width override")
    ap.add_argument("--point", default="", help="schedule point (default: selector)")
    ap.add_argument("--p", type=int, default=256)
    ap.add_argument("--hw-block", type=int, default=0)
    ap.add_argument("--hw-variant", type=int, default=0)
    ap.add_argument("--sweep", default="", help="write the full candidate sweep (JSON) here")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-blocks", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    return ap.parse_args(argv)


def maybe_self_launch(args) -> None:
    """``--gpus N`` outside torchrun: re-run this script as N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    port = 29500 + (os.getpid() % 2000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dist_setup():
    """One process per GPU over NCCL.  SGAP_BENCH_SHARE_GPU=1 (a test hook for
    boxes with fewer GPUs than ranks) puts every rank on cuda:0 over gloo so
    the multi-rank path -- shards, barriers, max-over-ranks -- can run on one
    GPU; numbers from that mode are not scaling results."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("SGAP_BENCH_SHARE_GPU") == "1":
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def default_n(cfg: int) -> int:
    return {1: 32, 2: 128, 3: 64, 4: 128, 5: 128}[cfg]


def build_workload(cfg: int, world: int, seed: int, device, weak: bool = False):
    from paper_2209_02882_b200 import generators as G
    if cfg == 2 and weak:
        scale = 20 + int(round(math.log2(world)))
        g = G.rmat(scale, 16, seed=seed, device=device)
        desc = f"config 2 weak: R-MAT scale {scale}, edge factor 16, permuted" + \
            (f" ({world}x config 2, {world} nnz-balanced row shards)" if world > 1 else "")
        return g, desc, "weak"
    g = G.config_matrix(cfg, device=device, seed=seed)
    desc = f"config {cfg}: {g.label}" + \
        (f" ({world} nnz-balanced row shards, B replicated)" if world > 1 else "")
    return g, desc, "strong"


def dense_b(num_rows: int, n: int, seed: int, device) -> torch.Tensor:
    gen = torch.Generator(device=device)
    gen.manual_seed(seed + 1)
    return (torch.rand((num_rows, n), generator=gen, dtype=torch.float32, device=device) * 2.0 - 1.0)


class ClockSampler:
    """NVML clock/throttle sampling in a thread during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clocks": 0x100,
    }

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML unavailable
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self) -> dict:
        names = [k for k, bit in self.REASONS.items() if self.reasons & bit and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def host_threads() -> int:
    """All cores this process may run on (torchrun sets OMP_NUM_THREADS=1 for
    multi-rank jobs; the CPU baseline deliberately uses every core)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def measured_peaks() -> dict:
    """HBM GB/s from MEASURED_PEAKS.json (driver-written); the FP32 FMA peak
    is not measured there, so it is the nominal 148 SMs x 128 lanes x 2 FLOP
    at the recorded max SM clock."""
    out = {"hbm_gbs": FALLBACK_HBM_GBS, "hbm_source": "fallback (B200_PROFILING.md)",
           "sm_mhz": 1965.0}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            rec = json.loads(p.read_text())
            out["hbm_gbs"] = float(rec["hbm_gbs"])
            out["hbm_source"] = "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
            out["sm_mhz"] = float(rec.get("sm_max_mhz", 1965.0))
        except Exception:
            pass
    out["fp32_tflops"] = SMS * FP32_LANES_PER_SM * 2 * out["sm_mhz"] * 1e6 / 1e12
    out["fp32_source"] = f"nominal: {SMS} SMs x {FP32_LANES_PER_SM} FMA lanes x 2 at {out['sm_mhz']:.0f} MHz"
    return out


def algorithmic_bytes(m: int, nnz: int, n: int, touched: int, esz: int = 4) -> int:
    """A streamed once (row_ptr + int32 col + fp32 val), each
    touched B row read once, C written once."""
    return 4 * (m + 1) + 8 * nnz + esz * n * touched + esz * m * n


def roofline(m: int, nnz: int, n: int, touched: int, kernel_ms: float, peaks: dict) -> dict:
    """t_roof = max(bytes / BW_HBM, 2 nnz N / P_FP32);
    frac = t_roof / t_measured.  ``achieved``/``peak`` are stated in the unit
    of the bound that binds."""
    abytes = algorithmic_bytes(m, nnz, n, touched)
    flops = 2.0 * nnz * n
    t_hbm = abytes / (peaks["hbm_gbs"] * 1e9)
    t_fma = flops / (peaks["fp32_tflops"] * 1e12)
    t = kernel_ms * 1e-3
    if t_hbm >= t_fma:
        r = {"bound": "hbm", "achieved": abytes / t / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    else:
        r = {"bound": "fp32_fma", "achieved": flops / t / 1e12, "peak": peaks["fp32_tflops"],
             "unit": "TFLOP/s"}
    r["frac"] = max(t_hbm, t_fma) / t
    r.update({"algorithmic_bytes": abytes, "t_hbm_ms": t_hbm * 1e3, "t_fp32_ms": t_fma * 1e3,
              "hbm_frac": t_hbm / t, "fp32_frac": t_fma / t, "kernel_ms": kernel_ms,
              "peak_source": {"hbm": peaks["hbm_source"], "fp32": peaks["fp32_source"]}})
    return r


def ncu_traffic(workload: str, point: str, hw_variant: int):
    """dram read+write bytes per launch of the dominant kernel from the
    committed ncu --set full capture of this build (profiles/ncu_traffic.json,
    written by tools/ncu_traffic.py), when one exists for this workload."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        rec = json.loads(p.read_text())

        def same_kernel(a: str, b: str) -> bool:
            # the shifted-block walk (row-multiple variant 8) ignores g: every
            # row:g point with the same c runs the same kernel
            if a == b:
                return True
            return (hw_variant == 8 and a.startswith("row:") and b.startswith("row:")
                    and "/" not in a.split(",")[0] and "/" not in b.split(",")[0]
                    and a.split(",")[1:] == b.split(",")[1:])

        for r in rec.get("entries", []):
            if (r.get("workload") == workload and same_kernel(r.get("point", ""), point)
                    and int(r.get("hw_variant", 0)) == hw_variant):
                return {"bytes": r.get("dram_bytes"), "kernel": r.get("kernel"),
                        "captured": r.get("captured"), "source": "profiles/ncu_traffic.json"}
    except Exception:
        return None
    return None


# --------------------------------------------------------------------------- CPU baselines

def _ref_import():
    """The reference package installed from /root/reference into baseline/_ref
    (pip --target; travels to the GPU box).  None when absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "spmmlab").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from spmmlab import matrices as M  # noqa: F401
        return M
    except Exception:
        return None


_W = {}


def _ref_worker_init(rp, ci, vals, bsub, n):
    """One row slice of the sample as the reference's own CsrMatrix /
    DenseMatrix (columns remapped onto the slice's touched B rows, which
    changes no product or summation order)."""
    M = _ref_import()
    uniq, inv = np.unique(ci, return_inverse=True)
    _W["a"] = M.CsrMatrix(len(rp) - 1, len(uniq), rp.astype(np.int64), inv.astype(np.int64),
                          vals.astype(np.float64))
    _W["b"] = M.DenseMatrix(len(uniq), n, np.ascontiguousarray(bsub[uniq], dtype=np.float64).reshape(-1))
    _W["oracle"] = M.dense_spmm_oracle


def _ref_worker_run(_):
    c = _W["oracle"](_W["a"], _W["b"])
    return float(c.vals[:8].sum())


def reference_cpu(rp, ci, vals, b_host, n, *, workers: int, nnz_per_worker: int, steps: int,
                  warmup: int):
    """The reference's CPU path (spmmlab.matrices.dense_spmm_oracle, pure
    Python over nonzeros, numpy over the N columns) on ``workers`` processes,
    each on its own contiguous row slice of the leading rows of the workload.
    Returns (GFLOP/s, seconds per step, sample description)."""
    import multiprocessing as mp
    total = min(int(rp[-1]), nnz_per_worker * workers)
    r_end = max(1, min(int(np.searchsorted(rp, total, side="left")), len(rp) - 1))
    s_nnz = int(rp[r_end])
    cuts = np.searchsorted(rp[: r_end + 1], np.linspace(0, s_nnz, workers + 1), side="left")
    cuts[0], cuts[-1] = 0, r_end
    slices = []
    for w in range(workers):
        lo, hi = int(cuts[w]), int(cuts[w + 1])
        if hi <= lo:
            continue
        p0, p1 = int(rp[lo]), int(rp[hi])
        slices.append((rp[lo:hi + 1] - p0, ci[p0:p1], vals[p0:p1]))
    ctx = mp.get_context("fork")
    pools = [ctx.Pool(1, initializer=_ref_worker_init, initargs=(s[0], s[1], s[2], b_host, n))
             for s in slices]
    try:
        def one_step():
            rs = [p.apply_async(_ref_worker_run, (0,)) for p in pools]
            for r in rs:
                r.get()
        for _ in range(warmup):
            one_step()
        t0 = time.perf_counter()
        for _ in range(steps):
            one_step()
        dt = (time.perf_counter() - t0) / steps
    finally:
        for p in pools:
            p.terminate()
    value = 2.0 * s_nnz * n / dt / 1e9
    sample = (f"spmmlab.matrices.dense_spmm_oracle (the reference, pure Python, baseline/_ref) on "
              f"rows [0, {r_end}) = {s_nnz} nnz x N={n} per step, {len(slices)} processes x 1 "
              "core, each on a contiguous row slice")
    return value, dt, sample, len(slices)


def port_cpu(rp, ci, vals, b_host, n, *, threads: int, sample_nnz: int, reps: int):
    """The oracle's C restatement of dense_spmm_oracle (bit-identical f64,
    OpenMP) on ``threads`` cores over the leading rows holding ~sample_nnz."""
    import oracle
    r_end = max(1, min(int(np.searchsorted(rp, min(int(rp[-1]), sample_nnz), side="left")),
                       len(rp) - 1))
    srp = rp[: r_end + 1].astype(np.int32)
    s_nnz = int(srp[-1])
    oracle.spmm_f64(srp, ci[:s_nnz], vals[:s_nnz], b_host, n, threads=threads)
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.spmm_f64(srp, ci[:s_nnz], vals[:s_nnz], b_host, n, threads=threads)
    dt = (time.perf_counter() - t0) / reps
    return (2.0 * s_nnz * n / dt / 1e9,
            f"oracle/ (C fp64 port of dense_spmm_oracle, OpenMP) on rows [0, {r_end}): "
            f"{s_nnz} nnz x N={n}, {reps} reps")


# --------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """``--impl reference``: the reference's own CPU implementation of the
    path (spmmlab's dense_spmm_oracle from baseline/_ref) on this host's
    cores, on a bounded sample of the same workload; rank 0 only.  Falls back
    to the oracle's C port (kind "port") when baseline/_ref is absent."""
    if rank != 0:
        return
    cfg = args.config
    n = args.n or default_n(cfg)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g, desc, scaling = build_workload(cfg, 1, args.seed, dev, weak=args.weak)
    rp = g.row_ptr.cpu().numpy().astype(np.int64)
    ci = g.col_idx.cpu().numpy().astype(np.int32)
    vals = g.vals.cpu().numpy().astype(np.float32)
    b_host = dense_b(g.num_cols, n, args.seed, dev).cpu().numpy()
    cores = host_threads()
    if _ref_import() is not None:
        workers = max(1, min(cores, 32))
        value, dt, sample, used = reference_cpu(rp, ci, vals, b_host, n, workers=workers,
                                                nnz_per_worker=150_000, steps=args.steps,
                                                warmup=min(args.warmup, 1))
        kind = "reference"
    else:
        value, sample = port_cpu(rp, ci, vals, b_host, n, threads=cores, sample_nnz=4_000_000,
                                 reps=args.steps)
        dt = 2.0 * 4_000_000 * n / value / 1e9
        used, kind = cores, "port"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "rows": g.num_rows, "nnz": g.nnz, "n": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": kind,
                         "sample": sample, "host_cores": cores},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm

def main():
    args = parse_args()
    maybe_self_launch(args)
    rank, world, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    from paper_2209_02882_b200.device import DeviceCsr, launches_per_call, prepare_aux, spmm
    from paper_2209_02882_b200.partition import plan_shards, shard_csr
    from paper_2209_02882_b200.selector import (Candidate, autotune, candidates, heuristic,
                                                matrix_stats, plan_for, refine)
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = args.config
    n = args.n or default_n(cfg)
    g, desc, scaling = build_workload(cfg, world, args.seed, dev, weak=args.weak)
    total_nnz = g.nnz
    plan = plan_shards(g.row_ptr.cpu().numpy(), world)
    rp, ci, vals = shard_csr(g.row_ptr, g.col_idx, g.vals, plan, rank)
    lo, hi = plan.rows(rank)
    a = DeviceCsr(hi - lo, g.num_cols, rp.to(torch.int32).contiguous(),
                  ci.to(torch.int32).contiguous(), vals.to(torch.float32).contiguous())
    del rp, ci, vals, g
    torch.cuda.empty_cache()
    touched = int(torch.unique(a.col_idx).numel()) if a.nnz else 0
    rp_host = a.row_ptr.cpu().numpy().astype(np.int64)
    b = dense_b(a.num_cols, n, args.seed, dev)
    c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    stats = matrix_stats(rp_host, a.num_cols)

    # ---- schedule choice (untimed)
    sweep_rows = []
    if args.point:
        choice = Candidate(args.point, args.p, args.hw_block, args.hw_variant)
    else:
        choice = None
        if rank == 0:
            ranked = autotune(a, b, c, n, candidates(n), reps=2, row_ptr_host=rp_host,
                              stream=stream, max_ms=50.0)
            sweep_rows = [{"point": cd.point, "p": cd.p, "hw_variant": cd.hw_variant, "ms": ms,
                           "gflops": 2.0 * a.nnz * n / (ms * 1e6)} for cd, ms in ranked]
            # the leaders again, interleaved (drift-proof pick among near-ties)
            final = refine(a, b, c, n, ranked, row_ptr_host=rp_host, stream=stream)
            choice = final[0][0]
        if world > 1:
            obj = [choice]
            dist.broadcast_object_list(obj, src=0)
            choice = obj[0]
    heur = heuristic(stats, n)
    k = plan_for(choice, n, a.num_rows, a.num_cols, rp_host)
    aux = prepare_aux(k, a, stream=stream)

    def step():
        spmm(k, a, b, c, aux=aux, hw_block=choice.hw_block, hw_variant=choice.hw_variant,
             stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = starts[0].elapsed_time(ends[-1])
    per_step = [starts[i].elapsed_time(ends[i]) for i in range(args.steps)]
    kernel_ms = statistics.mean(per_step)
    rank_ms = [total_ms]
    if world > 1:
        rank_ms = [None] * world
        dist.all_gather_object(rank_ms, total_ms)
    total_ms = max(rank_ms)  # max over ranks
    ms_per_step = total_ms / args.steps
    value = 2.0 * total_nnz * n / (ms_per_step * 1e6)

    # ---- roofline of the SpMM call (this rank's shard)
    peaks = measured_peaks()
    roof = roofline(a.num_rows, a.nnz, n, touched, kernel_ms, peaks)
    roof["kernel_ms_covers"] = ("the whole SpMM call (zero-fill + main kernel + long-row fold), "
                                "CUDA events on the launch stream, mean over the timed steps")
    roof["kernel_ms_median"] = statistics.median(per_step)
    roof["kernel_share"] = kernel_ms / ms_per_step
    workload_key = f"cfg{cfg}:world{world}:n{n}" + (":weak" if args.weak else "")
    roof["traffic"] = None
    tr = ncu_traffic(workload_key, choice.point, choice.hw_variant)
    if tr is not None:
        roof["traffic"] = tr["bytes"]
        roof["traffic_info"] = tr
        if tr["bytes"]:
            roof["traffic_over_algorithmic"] = tr["bytes"] / roof["algorithmic_bytes"]
            # the DRAM bytes that actually move, against the same measured peak:
            # how close the walk runs to the bandwidth floor of its access order
            roof["traffic_gbs"] = tr["bytes"] / (kernel_ms * 1e-3) / 1e9
            roof["traffic_frac_of_peak"] = roof["traffic_gbs"] / peaks["hbm_gbs"]
    roof["b_gather_bytes"] = a.nnz * n * 4  # every nonzero gathers a whole B row through L2
    roof["b_gather_tbs"] = roof["b_gather_bytes"] / (kernel_ms * 1e-3) / 1e12

    # ---- the optional collectives around the shard-parallel SpMM:
    # B replication (NCCL broadcast over NVLink) and the C gather to rank 0
    # (ncclSend/ncclRecv of unequal row slabs) -- set-up and epilogue, timed
    # separately, never inside ``value``
    collectives = None
    if world > 1 and os.environ.get("SGAP_BENCH_SHARE_GPU") != "1":
        collectives = time_collectives(b, c, plan, rank, dev, stream)
    # ---- end to end through host buffers
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, a, b, c, k, choice, plan_for, n, total_nnz, world, dev, stream)

    # ---- one call through the reference-facing drop-in (sim.run on host
    # CsrMatrix / DenseMatrix in the reference's float64 layout)
    if e2e is not None and rank == 0 and world == 1:
        e2e["dropin"] = measure_dropin(a, b, k, n)

    # ---- CPU baselines (rank 0, single GPU only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = host_threads()
        h_ci32 = a.col_idx.cpu().numpy()
        h_v32 = a.vals.cpu().numpy()
        h_b32 = b.cpu().numpy()
        pv, psample = port_cpu(rp_host, h_ci32, h_v32, h_b32, n, threads=threads,
                               sample_nnz=4_000_000, reps=3)
        cpu = {"value": pv, "unit": UNIT, "cores": threads, "kind": "port", "sample": psample}
        if _ref_import() is not None:
            rv, _, rsample, _ = reference_cpu(rp_host, h_ci32, h_v32, h_b32, n, workers=1,
                                              nnz_per_worker=150_000, steps=2, warmup=0)
            cpu["reference_1core"] = {"value": rv, "unit": UNIT, "cores": 1, "kind": "reference",
                                      "sample": rsample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": desc, "rows": int(plan.starts[-1]), "nnz": total_nnz, "n": n,
                "shard_rows": a.num_rows, "shard_nnz": a.nnz, "touched_b_rows": touched,
                "schedule": choice.point, "p": choice.p, "hw_variant": choice.hw_variant,
                "family": k.family, "heuristic_choice": heur.label(),
                "selector": "given" if args.point else "autotune",
                "parallelism": f"row-shard{world}" if world > 1 else "single",
                "shard_row_starts": [int(x) for x in plan.starts] if world > 1 else None,
                "rank_total_ms": rank_ms if world > 1 else None,
                "l2": "inputs > L2 (A+B+C far above 126 MB): no flush needed",
                "plan": {"table_rows": aux.table_rows, "longest_row": aux.longest_row,
                         "exact_rows": aux.exact_count, "workspace_bytes": aux.nbytes()},
                "stats": stats.as_dict(),
            },
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "collectives": collectives,
            "gpu_launches": args.steps * launches_per_call(k, aux, hw_variant=choice.hw_variant),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
        if args.sweep and sweep_rows:
            Path(args.sweep).parent.mkdir(parents=True, exist_ok=True)
            Path(args.sweep).write_text(json.dumps({"workload": desc, "n": n, "rows": sweep_rows,
                                                    "heuristic": heur.label()}, indent=1))
    if world > 1:
        dist.destroy_process_group()


def time_collectives(b, c, plan, rank, dev, stream):
    """B broadcast from rank 0 and the C row-slab gather to rank 0 over the
    process group (NCCL on the GPU box), CUDA events, max over ranks."""
    import torch.distributed as dist
    from paper_2209_02882_b200.parallel import broadcast_dense, gather_rows

    def timed(fn):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    timed(lambda: broadcast_dense(b, src=0))  # warm the communicator
    t_bc, _ = timed(lambda: broadcast_dense(b, src=0))
    t_ga, full = timed(lambda: gather_rows(c, plan, root=0))
    del full
    bb = b.numel() * b.element_size()
    cb = int(plan.starts[-1]) * c.shape[1] * c.element_size()
    return {"broadcast_b_ms": t_bc, "broadcast_b_bytes": bb,
            "broadcast_b_gbs": bb / (t_bc * 1e-3) / 1e9,
            "gather_c_ms": t_ga, "gather_c_bytes": cb, "gather_c_gbs": cb / (t_ga * 1e-3) / 1e9,
            "backend": dist.get_backend(),
            "note": "set-up (B replica) and optional epilogue (C on rank 0); not part of value"}


def measure_dropin(a, b, k, n):
    """One SpMM through ``paper_2209_02882_b200.sim.run(kernel, CsrMatrix,
    DenseMatrix, precision="single")`` -- the call a reference caller makes
    (spmmlab/sim.py:431-487): float64 host operands in, float64 host C out,
    conversions, uploads, validation, planning and the download all inside
    the wall-clock region.  Skipped when the host lacks the memory for the
    reference layout (~2x the float32 footprint)."""
    from paper_2209_02882_b200.matrices import CsrMatrix, DenseMatrix
    from paper_2209_02882_b200.sim import run as sim_run
    need = (a.nnz * 16 + a.num_cols * n * 8 + a.num_rows * n * 8) * 3
    try:
        import psutil
        if psutil.virtual_memory().available < need:
            return {"skipped": f"needs ~{need / 1e9:.0f} GB host memory"}
    except Exception:
        pass
    A = CsrMatrix(a.num_rows, a.num_cols, a.row_ptr.cpu().numpy().astype(np.int64),
                  a.col_idx.cpu().numpy().astype(np.int64),
                  a.vals.cpu().numpy().astype(np.float64))
    B = DenseMatrix(a.num_cols, n, b.cpu().numpy().astype(np.float64).reshape(-1))
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    C, m = sim_run(k, A, B, precision="single")
    wall = time.perf_counter() - t0
    out = {"wall_ms": wall * 1e3, "gflops": 2.0 * a.nnz * n / wall / 1e9,
           "kernel_ms": m.device_ms, "h2d_bytes": A.nnz * 8 + (A.num_rows + 1) * 4 + B.vals.size * 4,
           "d2h_bytes": C.vals.size * 4,
           "path": "sim.run(kernel, CsrMatrix f64, DenseMatrix f64, precision='single'): host "
                   "f64->f32 / int64->int32 conversion, upload, CSR validation, sgap_plan, SpMM, "
                   "download, f32->f64; one call, wall clock"}
    del A, B, C
    return out


def measure_e2e(args, a, b, c, k, choice, plan_for, n, total_nnz, world, dev, stream):
    """The same metric through host buffers: (1) steady state through
    ``pipeline.HostSpmm`` (pinned A, B up / SpMM / C down per step,
    overlapped); (2) one cold start through the public device API: upload A
    and B, plan on the device (sgap_plan), SpMM, download C."""
    import torch.distributed as dist
    from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm
    from paper_2209_02882_b200.pipeline import HostSpmm
    h_rp = a.row_ptr.cpu().pin_memory()
    h_ci = a.col_idx.cpu().pin_memory()
    h_v = a.vals.cpu().pin_memory()
    h_b = b.cpu().pin_memory()
    h_c = torch.empty(c.shape, dtype=c.dtype).pin_memory()

    def plan_block(rows, sub_rp):
        return plan_for(choice, n, rows, a.num_cols, sub_rp)

    pipe = HostSpmm(a.num_rows, a.num_cols, n, h_rp, h_ci, plan_block, blocks=args.e2e_blocks,
                    hw_variant=choice.hw_variant)
    pipe(h_v, h_b, h_c)
    pipe.wait()
    torch.cuda.synchronize()
    e_steps = max(3, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e_steps):
        pipe(h_v, h_b, h_c)
    pipe.wait(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    h2d, d2h = pipe.h2d_bytes(), pipe.d2h_bytes()
    del pipe
    torch.cuda.empty_cache()
    # the PCIe floor of one step: the same bytes up and down at once, no compute
    s_up, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    d_rp, d_ci, d_v = (torch.empty_like(x, device=dev) for x in (h_rp, h_ci, h_v))
    d_c = torch.empty_like(h_c, device=dev)

    def copies():
        s_up.wait_stream(stream)
        s_dn.wait_stream(stream)
        with torch.cuda.stream(s_up):
            for dst, src in ((d_rp, h_rp), (d_ci, h_ci), (d_v, h_v), (b, h_b)):
                dst.copy_(src, non_blocking=True)
        with torch.cuda.stream(s_dn):
            h_c.copy_(d_c, non_blocking=True)
        stream.wait_stream(s_up)
        stream.wait_stream(s_dn)

    floor = float("inf")
    for _ in range(3):
        e0.record(stream)
        copies()
        e1.record(stream)
        e1.synchronize()
        floor = min(floor, e0.elapsed_time(e1))
    del d_c
    # cold start: upload + device planning + SpMM + download, serial
    torch.cuda.synchronize()
    e0.record(stream)
    d_rp.copy_(h_rp, non_blocking=True)
    d_ci.copy_(h_ci, non_blocking=True)
    d_v.copy_(h_v, non_blocking=True)
    b.copy_(h_b, non_blocking=True)
    a2 = DeviceCsr(a.num_rows, a.num_cols, d_rp, d_ci, d_v)
    aux2 = prepare_aux(k, a2, stream=stream)
    spmm(k, a2, b, c, aux=aux2, hw_block=choice.hw_block, hw_variant=choice.hw_variant,
         stream=stream)
    h_c.copy_(c, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    cold_ms = e0.elapsed_time(e1)
    del aux2, a2, d_rp, d_ci, d_v
    ms = float(te.item())
    return {"value": 2.0 * total_nnz * n / (ms * 1e6), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": ms, "steps": e_steps,
            "pcie_floor_ms": floor, "frac_of_pcie_floor": floor / ms,
            "cold_start_ms": cold_ms,
            "cold_start_gflops": 2.0 * a.nnz * n / (cold_ms * 1e6),
            "cold_start_path": "pinned host A, B -> device; sgap_plan (row stats, block starts, "
                               "row ids, float64 table) -> SpMM -> C to pinned host, one stream",
            "path": f"pinned host A,B -> {args.e2e_blocks} row blocks: H2D / SpMM / D2H C "
                    "overlapped on 3 streams, device buffers double-buffered across steps "
                    "(paper_2209_02882_b200.pipeline.HostSpmm; structure planned once)"}


if __name__ == "__main__":
    main()
