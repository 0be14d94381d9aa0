"""Generate the golden fixtures by importing the reference package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py            # fast fixtures
    python tests/golden/make_golden.py --cfg1-sim # + slow config-1 simulator pins

The reference (``spmmlab``) is pure Python; it cannot travel to the GPU box,
so its outputs are frozen here as small fixtures.  Nothing in the product or
in the ``-m gpu`` tests reads ``/root/reference`` at run time.

Fixtures:
  space.json           enumerate_space / enumerate_report / lowering geometry
                       (grid, block, block_starts) for many (n, p) configs
  zoo_oracle.npz       dense_spmm_oracle outputs on the conftest matrix zoo
  sim_metrics.json     sim.run atomic_ops + max_rel_error for every templated
                       point on the zoo at n in {4, 8}, p = 256
  sim_long.json        sim.run atomic_ops for long chunks (nnz:g with g in
                       64..512, all walks' writeback logic) on three
                       matrices with ~20-40k nonzeros incl. power-law rows
  group_primitives.npz exec_seg_reduce_group / exec_atomic_add_group cases
  cfg1.json            config-1 input/oracle hashes (+ simulator pins with
                       --cfg1-sim)
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent

sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

from spmmlab import lowering as ref_lowering  # noqa: E402
from spmmlab.lowering import KernelConfig, compute_block_starts  # noqa: E402
from spmmlab.matrices import CsrMatrix, dense_spmm_oracle, random_csr, random_dense  # noqa: E402
from spmmlab.runner import build_kernel, enumerate_report, verify_point  # noqa: E402
from spmmlab.sim import exec_atomic_add_group, exec_seg_reduce_group, run  # noqa: E402
from spmmlab.space import da_spmm_points, enumerate_space, parse_point  # noqa: E402
from spmmlab.templates import algorithm_template  # noqa: E402

from conftest import matrix_zoo  # noqa: E402  (reference test fixtures)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CONFIGS = [
    (4, 256), (8, 256), (16, 256), (32, 256), (32, 1024), (64, 256),
    (128, 256), (128, 1024), (256, 256), (512, 256), (1, 32), (3, 96),
    (12, 128), (6, 64), (128, 4096), (2, 64),
]

GEOM_MATRICES = {
    "emit64": lambda: random_csr(64, 64, 0.0625, seed=1),
    "dense96": lambda: random_csr(96, 96, 0.5, seed=3),
    "tall300": lambda: random_csr(300, 16, 0.1, seed=4),
    "empty16": lambda: CsrMatrix(16, 16, np.zeros(17, dtype=np.int64), [], []),
    "lead_empty": lambda: CsrMatrix(6, 4, [0, 0, 0, 2, 2, 5, 5], [0, 3, 0, 1, 2], [1.0] * 5),
}


def make_space():
    enum = enumerate_space()
    out = {
        "legal": [str(p) for p in enum.legal],
        "rejected": {str(p): r for p, r in enum.rejected},
        "da_spmm": [str(p) for p in da_spmm_points()],
        "configs": {},
    }
    mats = {k: f() for k, f in GEOM_MATRICES.items()}
    for n, p in CONFIGS:
        cfg = KernelConfig(n=n, p=p)
        rep = enumerate_report(cfg)
        entry = {"templated": [e["point"] for e in rep["legal"] if e["templated"]],
                 "families": {e["point"]: e["family"] for e in rep["legal"]},
                 "kernels": {}}
        for ptxt in entry["templated"]:
            per = {}
            for mname, mat in mats.items():
                k = build_kernel(parse_point(ptxt), cfg, mat)
                rec = {"grid": k.grid_size, "block": k.block_size, "name": k.name,
                       "family": k.family}
                if k.block_starts is not None:
                    rec["starts_len"] = int(len(k.block_starts))
                    rec["starts_sha"] = sha(np.asarray(k.block_starts, np.int64))
                    if mname in ("emit64", "lead_empty", "empty16"):
                        rec["starts"] = [int(x) for x in k.block_starts]
                per[mname] = rec
            entry["kernels"][ptxt] = per
        out["configs"][f"{n},{p}"] = entry
    # compute_block_starts / binary_search_before known answers on random rows
    rng = np.random.default_rng(1234)
    cases = []
    for _ in range(200):
        rows = int(rng.integers(1, 40))
        counts = rng.integers(0, 6, size=rows)
        rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        nnz = int(rp[-1])
        chunk = int(rng.integers(1, 20))
        nb = -(-nnz // chunk) if nnz else 0
        starts = compute_block_starts(rp, chunk, nb)
        lo = int(rng.integers(0, rows))
        hi = int(rng.integers(lo, rows + 1))
        tgt = int(rng.integers(-2, nnz + 3))
        cases.append({"row_ptr": rp.tolist(), "chunk": chunk, "num_blocks": nb,
                      "starts": starts.tolist(), "lo": lo, "hi": hi, "target": tgt,
                      "search": int(ref_lowering.binary_search_before(rp, lo, hi, tgt))})
    out["starts_cases"] = cases
    (OUT / "space.json").write_text(json.dumps(out, sort_keys=True))
    print("space.json", len(out["legal"]), len(out["rejected"]))


def make_zoo():
    arrays = {}
    meta = []
    for label, mat, b_seed in matrix_zoo():
        for n in (4, 8):
            b = random_dense(mat.num_cols, n, seed=b_seed)
            c = dense_spmm_oracle(mat, b)
            key = f"{label}|{n}"
            arrays[key] = c.vals
        meta.append({"label": label, "rows": mat.num_rows, "cols": mat.num_cols,
                     "b_seed": b_seed, "row_ptr_sha": sha(mat.row_ptr),
                     "col_idx_sha": sha(mat.col_idx), "vals_sha": sha(mat.vals)})
    np.savez_compressed(OUT / "zoo_oracle.npz", **arrays)
    (OUT / "zoo_meta.json").write_text(json.dumps(meta, indent=1))
    print("zoo_oracle.npz", len(arrays))


def make_sim_metrics():
    t0 = time.time()
    rows = []
    for n in (4, 8):
        cfg = KernelConfig(n=n, p=256)
        templated = [p for p in enumerate_space().legal if algorithm_template(p, cfg) is not None]
        for label, mat, b_seed in matrix_zoo():
            b = random_dense(mat.num_cols, n, seed=b_seed)
            for pt in templated:
                rep = verify_point(mat, pt, cfg, b=b)
                rows.append({"matrix": label, "n": n, "p": 256, "point": str(pt),
                             "family": rep.family, "grid": rep.grid_size,
                             "block": rep.block_size,
                             "atomic_ops": rep.metrics.atomic_ops,
                             "max_rel_error": rep.max_rel_error})
    (OUT / "sim_metrics.json").write_text(json.dumps(rows))
    print("sim_metrics.json", len(rows), f"{time.time() - t0:.1f}s")


def make_group_primitives():
    rng = np.random.default_rng(97)
    arrays = {}
    for gsz in (1, 2, 4, 8, 16, 32):
        groups = 256
        lanes = groups * gsz
        val = rng.uniform(-1.0, 1.0, size=lanes)
        active = rng.random(lanes) < 0.8
        idx_same = np.repeat(rng.integers(0, 512, size=groups), gsz)
        out = np.zeros(512)
        nwb = exec_atomic_add_group(idx_same, val, out, active, group_size=gsz)
        arrays[f"atomic|{gsz}|idx"] = idx_same
        arrays[f"atomic|{gsz}|val"] = val
        arrays[f"atomic|{gsz}|active"] = active
        arrays[f"atomic|{gsz}|out"] = out
        arrays[f"atomic|{gsz}|wb"] = np.array([nwb])
        idx_sorted = np.sort(rng.integers(0, 512, size=(groups, gsz)), axis=1).ravel()
        out = np.zeros(512)
        nwb = exec_seg_reduce_group(idx_sorted, val, out, active, group_size=gsz)
        arrays[f"seg|{gsz}|idx"] = idx_sorted
        arrays[f"seg|{gsz}|val"] = val
        arrays[f"seg|{gsz}|active"] = active
        arrays[f"seg|{gsz}|out"] = out
        arrays[f"seg|{gsz}|wb"] = np.array([nwb])
    np.savez_compressed(OUT / "group_primitives.npz", **arrays)
    print("group_primitives.npz", len(arrays))


def make_cfg1(with_sim: bool):
    a = random_csr(4096, 4096, 0.01, seed=1)
    b = random_dense(4096, 32, seed=2)
    c = dense_spmm_oracle(a, b)
    a32 = CsrMatrix(a.num_rows, a.num_cols, a.row_ptr, a.col_idx,
                    a.vals.astype(np.float32).astype(np.float64))
    b32 = type(b)(b.num_rows, b.num_cols, b.vals.astype(np.float32).astype(np.float64))
    c32 = dense_spmm_oracle(a32, b32)
    out = {"nnz": a.nnz, "row_ptr_sha": sha(a.row_ptr), "col_idx_sha": sha(a.col_idx),
           "vals_sha": sha(a.vals), "b_sha": sha(b.vals), "oracle_sha": sha(c.vals),
           "oracle_f32in_sha": sha(c32.vals),
           "oracle_rows_0_3": c.vals[: 4 * 32].tolist(), "sim": []}
    path = OUT / "cfg1.json"
    if not with_sim and path.exists():
        out["sim"] = json.loads(path.read_text()).get("sim", [])
    if with_sim:
        for ptxt, p in (("row:1,col:1,r:1", 1024), ("nnz:32,col:1,r:1", 1024),
                        ("row:1/32,col:1,r:32", 1024), ("nnz:1,col:1,r:32", 1024),
                        ("nnz:1,col:4,r:8", 256), ("row:1/4,col:4,r:4", 256)):
            cfg = KernelConfig(n=32, p=p)
            k = build_kernel(parse_point(ptxt), cfg, a)
            t0 = time.time()
            got, m = run(k, a, b, precision="single")
            dt = time.time() - t0
            err = float(np.max(np.abs(got.vals - c.vals) / (np.abs(c.vals) + 1)))
            out["sim"].append({"point": ptxt, "p": p, "grid": k.grid_size,
                               "block": k.block_size, "atomic_ops": m.atomic_ops,
                               "max_rel_error_single": err, "sim_seconds": dt})
            print(ptxt, p, m.atomic_ops, err, f"{dt:.1f}s", flush=True)
    path.write_text(json.dumps(out, indent=1))
    print("cfg1.json")


def long_chunk_matrices():
    """Three matrices with enough nonzeros for several g = 512 chunks:
    uniform, power-law rows (hub rows span many chunks), and empty rows."""
    out = [("random:800x800:0.05:21", random_csr(800, 800, 0.05, seed=21))]
    rng = np.random.default_rng(22)
    m, k = 600, 3000
    lens = np.minimum((rng.pareto(1.2, m) * 8).astype(np.int64), 2500)
    lens[::7] = 0
    lens[3] = 2500
    rp = np.concatenate([[0], np.cumsum(lens)])
    cols = np.concatenate([np.sort(rng.choice(k, int(L), replace=False)) for L in lens if L])
    out.append(("powerlaw:600x3000:22", CsrMatrix(m, k, rp, cols, rng.uniform(-1, 1, rp[-1]))))
    lens = np.zeros(400, dtype=np.int64)
    lens[50:350] = rng.integers(0, 120, 300)
    rp = np.concatenate([[0], np.cumsum(lens)])
    cols = np.concatenate([np.sort(rng.choice(500, int(L), replace=False)) for L in lens if L])
    out.append(("gaps:400x500:22", CsrMatrix(400, 500, rp, cols, rng.uniform(-1, 1, rp[-1]))))
    return out


def make_sim_long():
    """Writeback counts of the reference simulator for long chunks (the
    bench's nnz:512 family member and its neighbours)."""
    t0 = time.time()
    rows = []
    n = 8
    cfg = KernelConfig(n=n, p=256)
    for label, mat in long_chunk_matrices():
        b = random_dense(mat.num_cols, n, seed=5)
        for g in (64, 128, 256, 512):
            for c in (1, 2, 4):
                pt = parse_point(f"nnz:{g},col:{c},r:1")
                k = build_kernel(pt, cfg, mat)
                if k is None:
                    continue
                got, m = run(k, mat, b)
                want = dense_spmm_oracle(mat, b)
                err = float(np.max(np.abs(got.vals - want.vals) / (np.abs(want.vals) + 1)))
                rows.append({"matrix": label, "n": n, "p": 256, "point": str(pt),
                             "grid": k.grid_size, "block": k.block_size, "nnz": mat.nnz,
                             "atomic_ops": m.atomic_ops, "max_rel_error": err,
                             "row_ptr_sha": sha(mat.row_ptr), "col_idx_sha": sha(mat.col_idx),
                             "vals_sha": sha(mat.vals)})
                print(label, pt, k.grid_size, m.atomic_ops, f"{time.time() - t0:.0f}s", flush=True)
    (OUT / "sim_long.json").write_text(json.dumps(rows, indent=1))
    print("sim_long.json", len(rows), f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg1-sim", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    todo = args.only.split(",") if args.only else ["space", "zoo", "sim", "groups", "cfg1"]
    if "space" in todo:
        make_space()
    if "zoo" in todo:
        make_zoo()
    if "groups" in todo:
        make_group_primitives()
    if "cfg1" in todo:
        make_cfg1(args.cfg1_sim)
    if "sim" in todo:
        make_sim_metrics()
    if "simlong" in todo:
        make_sim_long()
