"""Matrix Market ingest: host parser (matrices.loads_matrix_market, vectorised
numpy) vs the device path (ingest.load_matrix_market_device) on a generated
coordinate file; both results compared bit-for-bit."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2209_02882_b200.ingest import load_matrix_market_device  # noqa: E402
from paper_2209_02882_b200.matrices import loads_matrix_market  # noqa: E402

n_rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nnz = int(sys.argv[2]) if len(sys.argv) > 2 else 8_000_000
rng = np.random.default_rng(1)
r = rng.integers(1, n_rows + 1, nnz)
c = rng.integers(1, n_rows + 1, nnz)
for label, vals in (("6-digit values", np.char.mod("%.6e", rng.uniform(-1, 1, nnz))),
                    ("17-digit repr values", np.array([repr(float(x)) for x in rng.uniform(-1, 1, nnz)]))):
    body = np.char.add(np.char.add(np.char.add(r.astype(str), " "), np.char.add(c.astype(str), " ")), vals)
    text = f"%%MatrixMarket matrix coordinate real general\n{n_rows} {n_rows} {nnz}\n" + "\n".join(body) + "\n"
    t0 = time.time()
    host = loads_matrix_market(text)
    t_host = time.time() - t0
    load_matrix_market_device(text)  # warm (kernels, allocator)
    torch.cuda.synchronize()
    t0 = time.time()
    dev = load_matrix_market_device(text)
    torch.cuda.synchronize()
    t_dev = time.time() - t0
    same = (np.array_equal(dev.row_ptr.cpu().numpy(), host.row_ptr)
            and np.array_equal(dev.col_idx.cpu().numpy(), host.col_idx)
            and np.array_equal(dev.vals.cpu().numpy().view(np.int64), host.vals.view(np.int64)))
    print(f"{label}: {len(text) / 1e6:.0f} MB text, {nnz} entries: host {t_host:.2f} s, "
          f"device {t_dev:.2f} s ({t_host / t_dev:.1f}x), identical={same}", flush=True)
