"""Capture the DRAM traffic of the benched SpMM kernel at HEAD (the
``roofline.traffic`` figure of bench.py) and keep it under profiles/.

On the GPU box (one ncu --set full capture of the main kernel, after one
warm call):

    ncu --set full --clock-control none --import-source on \
        -k regex:'^(k_nnz_multiple|k_nnz_multiple_tma|k_nnz_multiple_staged|k_nnz_one|k_row_multiple|k_row_interleaved|k_row_staged|k_row_reciprocal)$' \
        --launch-skip 1 -c 1 -o gpurun_out/cap_cfg5 \
        python tools/ncu_traffic.py run --config 5 --point nnz:512,col:4,r:1 --p 256

Here (reads the report, updates profiles/ncu_traffic.json and writes the
summary next to it):

    python tools/ncu_traffic.py merge gpurun_out/cap_cfg5.ncu-rep --config 5 \
        --point nnz:512,col:4,r:1 --hw-variant 0 --summary profiles/r02_ncu_cfg5.json
"""
import argparse
import csv
import io
import json
import subprocess
import sys
from datetime import datetime, timezone
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))


def run(args):
    import numpy as np
    import torch
    import bench
    from paper_2209_02882_b200.device import DeviceCsr, prepare_aux, spmm
    from paper_2209_02882_b200.selector import Candidate, plan_for
    dev = torch.device("cuda", 0)
    n = args.n or bench.default_n(args.config)
    g, desc, _ = bench.build_workload(args.config, 1, 1, dev)
    a = DeviceCsr(g.num_rows, g.num_cols, g.row_ptr.to(torch.int32), g.col_idx.to(torch.int32),
                  g.vals.to(torch.float32))
    del g
    torch.cuda.empty_cache()
    b = bench.dense_b(a.num_cols, n, 1, dev)
    c = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
    rp = a.row_ptr.cpu().numpy().astype(np.int64)
    cand = Candidate(args.point, args.p, 0, args.hw_variant)
    k = plan_for(cand, n, a.num_rows, a.num_cols, rp)
    aux = prepare_aux(k, a)
    for _ in range(2):  # warm call (skipped by ncu), then the captured one
        spmm(k, a, b, c, aux=aux, hw_variant=args.hw_variant)
    torch.cuda.synchronize()
    print(desc, args.point, "variant", args.hw_variant)


def merge(args):
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    vals = rows[2]

    def get(name, scale_to_bytes=False):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        if scale_to_bytes:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[units[i]]
        return v

    dram = get("dram__bytes_read.sum", True) + get("dram__bytes_write.sum", True)
    kernel = vals[hdr.index("Kernel Name")][:120]
    n = args.n or {1: 32, 2: 128, 3: 64, 4: 128, 5: 128}[args.config]
    key = f"cfg{args.config}:world1:n{n}"
    path = ROOT / "profiles" / "ncu_traffic.json"
    doc = json.loads(path.read_text()) if path.exists() else {}
    doc["source"] = ("ncu --set full --clock-control none, one launch of the main SpMM kernel "
                     "after a warm call (tools/ncu_traffic.py); dram__bytes_read.sum + "
                     "dram__bytes_write.sum")
    ents = [e for e in doc.get("entries", [])
            if not (e.get("workload") == key and e.get("point") == args.point
                    and int(e.get("hw_variant", 0)) == args.hw_variant)]
    head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
                          cwd=str(ROOT)).stdout.strip()
    if not head:  # the GPU box has no .git: identify the build by the library hash
        import hashlib
        lib = ROOT / "paper_2209_02882_b200" / "libsgap.so"
        head = "libsgap.so sha256 " + hashlib.sha256(lib.read_bytes()).hexdigest()[:12]
    ents.append({"workload": key, "point": args.point, "hw_variant": args.hw_variant,
                 "kernel": kernel, "dram_bytes": int(dram),
                 "gpu_time_ms": get("gpu__time_duration.sum") / (1e6 if units[
                     hdr.index("gpu__time_duration.sum")] == "ns" else 1e3 if units[
                     hdr.index("gpu__time_duration.sum")] == "us" else 1),
                 "captured": f"{datetime.now(timezone.utc).date()} at {head}",
                 "report": Path(args.report).name})
    doc["entries"] = ents
    path.write_text(json.dumps(doc, indent=1))
    if args.summary:
        from ncu_summary import summarise
        Path(args.summary).write_text(json.dumps({"what": f"{key} {args.point} v{args.hw_variant}",
                                                  "captures": summarise(args.report)}, indent=1))
    print(key, args.point, kernel, f"{dram / 1e9:.3f} GB")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "merge"])
    ap.add_argument("report", nargs="?")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--point", default="nnz:512,col:4,r:1")
    ap.add_argument("--p", type=int, default=256)
    ap.add_argument("--hw-variant", type=int, default=0)
    ap.add_argument("--summary", default="")
    a = ap.parse_args()
    run(a) if a.mode == "run" else merge(a)
