"""Write a BASELINE config's CSR (int32 row_ptr/col_idx/row ids, float32 values)
as raw files <prefix>.rp/.ci/.av/.rid for the standalone walk probes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2209_02882_b200 import generators as g

dev = "cuda" if torch.cuda.is_available() else "cpu"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m = g.config_matrix(cfg, device=dev)
rp = m.row_ptr.to(torch.int64)
rid = torch.repeat_interleave(torch.arange(m.num_rows, device=rp.device), rp[1:] - rp[:-1])
for ext, t in (("rp", m.row_ptr.to(torch.int32)), ("ci", m.col_idx.to(torch.int32)),
               ("av", m.vals.to(torch.float32)), ("rid", rid.to(torch.int32))):
    t.cpu().numpy().tofile(f"{sys.argv[1]}.{ext}")
print(m.label, m.num_rows, int(rp[-1]))
