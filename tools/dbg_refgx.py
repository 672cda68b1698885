"""grad_X of one reference-precision step against the fp32 restatement (debug)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2510_11168_b200 as xmc
from oracle import lpxmc_oracle as O
from parity_util import torch_fp32_grad_x

L, k, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
B, D = 256, 768
g = torch.Generator(device="cuda"); g.manual_seed(7)
W0 = torch.empty((L, D), dtype=torch.float8_e4m3fn, device="cuda")
for r0 in range(0, L, 262_144):
    r1 = min(L, r0 + 262_144)
    W0[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, D), generator=g, device="cuda") * 0.02, xmc.E4M3)
rs = np.random.default_rng(3)
X = rs.normal(size=(B, D)).astype(np.float32)
si, li = O.synthetic_positives(L, B, 36.17, seed=4)
head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0.clone(), xmc.E4M3), num_chunks=k, precision=prec)
cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding="stochastic", sr_impl="hash")
gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(11), 0)
Xq = O.round_nearest(O.E4M3, X)
ref = torch_fp32_grad_x(W0, Xq, si, li)
err = (gx - ref).abs()
print(L, k, prec, "max abs err", float(err.max()), "ref max", float(ref.abs().max()), "rel", float(err.max() / ref.abs().max()))
