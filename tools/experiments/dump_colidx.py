"""Write config-2's col_idx (int32) in CSR order, plus the same indices sorted
(perfect-locality bound), for l2_gather_probe's file mode."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2209_02882_b200 import generators as g

dev = "cuda" if torch.cuda.is_available() else "cpu"
m = g.config_matrix(int(sys.argv[2]) if len(sys.argv) > 2 else 2, device=dev)
col = m.col_idx.to(torch.int32).cpu().numpy()
col.tofile(sys.argv[1] + ".csr")
np.sort(col).tofile(sys.argv[1] + ".sorted")
print(m.num_rows, col.size)
