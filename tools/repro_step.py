"""One head step of a given shape/precision (debug helper: run under compute-sanitizer)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11168_b200 as xmc
from oracle import lpxmc_oracle as O

L, B, fname, prec, k = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
impl = sys.argv[6] if len(sys.argv) > 6 else "splitmix64"
fmt = xmc.parse_format(fname)
g = torch.Generator(device="cuda"); g.manual_seed(17)
W0 = xmc.cast_native(torch.randn((L, 768), generator=g, device="cuda") * 0.02, fmt)
rs = np.random.default_rng(8)
X = rs.normal(size=(B, 768)).astype(np.float32)
si, li = O.synthetic_positives(L, B, 5.0, seed=9)
head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0, fmt), num_chunks=k, precision=prec)
cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic", sr_impl=impl)
gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(21), 3)
torch.cuda.synchronize()
print("ok", L, B, fname, prec, k, float(gx.abs().sum()))
