"""Freeze the reference compiler's emitted CUDA (spmmlab.cuda.emit_cuda,
cuda.py:91-183) for a set of schedule points, so the reference's own
fixed-schedule kernels can be compiled for sm_100a and timed on the B200 next
to ours (the "naive TACO" baseline).

Run in the build container (where /root/reference exists):

    python tests/golden/make_refgen.py

Writes tests/golden/refgen/manifest.json + one <id>.cu per distinct kernel
text.  The text is what the reference emits -- double precision, group macros
declared but not defined (cuda.py:52-56); baseline/refgen/ supplies the macro
bodies (sim.py:112-165 semantics) and instantiates each text at float32 and
float64.  Emission depends only on (point, n, p): the lowered body reads the
matrix through kernel arguments (grid_size/block_size are comments), checked
here by emitting every point against two different matrices.
"""

from __future__ import annotations

import hashlib
import json
import re
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "refgen"
sys.path.insert(0, str(REF_SRC))

from spmmlab.cuda import emit_cuda  # noqa: E402
from spmmlab.lowering import KernelConfig  # noqa: E402
from spmmlab.matrices import random_csr  # noqa: E402
from spmmlab.runner import build_kernel  # noqa: E402
from spmmlab.space import da_spmm_points, enumerate_space  # noqa: E402

CONFIGS = [(4, 256), (32, 256), (128, 256)]


def strip_comments(text: str) -> str:
    return "\n".join(l for l in text.splitlines() if not l.startswith("// grid_size")
                     and not l.startswith("// block_size"))


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    m1 = random_csr(64, 64, 0.0625, seed=1)
    m2 = random_csr(300, 200, 0.05, seed=7)
    corners = {str(p) for p in da_spmm_points()}
    entries, texts = [], {}
    for n, p in CONFIGS:
        cfg = KernelConfig(n=n, p=p)
        for point in enumerate_space().legal:
            k1 = build_kernel(point, cfg, m1)
            if k1 is None:
                continue
            k2 = build_kernel(point, cfg, m2)
            t1, t2 = emit_cuda(k1), emit_cuda(k2)
            assert strip_comments(t1) == strip_comments(t2), (str(point), n, p)
            body = strip_comments(t1)
            kid = hashlib.sha1(body.encode()).hexdigest()[:12]
            if kid not in texts:
                texts[kid] = body
                (OUT / f"{kid}.cu").write_text(body + "\n")
            name = re.search(r"__global__ void (\w+)\(", body).group(1)
            entries.append({"point": str(point), "n": n, "p": p, "family": k1.family,
                            "kernel": name, "id": kid, "block_size": k1.block_size,
                            "has_block_starts": k1.block_starts is not None,
                            "da_spmm_corner": str(point) in corners})
    (OUT / "manifest.json").write_text(json.dumps({"configs": CONFIGS, "kernels": entries},
                                                  indent=1) + "\n")
    print(f"{len(entries)} (point, n, p) entries, {len(texts)} distinct kernel texts")


if __name__ == "__main__":
    main()
