"""Debug: full-size shard linearity of grad_X (gxa + gxb vs gx1)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11168_b200 as xmc
from oracle import lpxmc_oracle as O

L, D, B = int(sys.argv[1]) if len(sys.argv) > 1 else 2_812_281, 768, 256
g = torch.Generator(device="cuda"); g.manual_seed(7)
W0 = torch.empty((L, D), dtype=torch.float8_e4m3fn, device="cuda")
for r0 in range(0, L, 262_144):
    r1 = min(L, r0 + 262_144)
    W0[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, D), generator=g, device="cuda") * 0.02, xmc.E4M3)
rs = np.random.default_rng(3)
X = rs.normal(size=(B, D)).astype(np.float32)
si, li = O.synthetic_positives(L, B, 36.17, seed=4)

def run(lo, hi, k=1, off=None, glob=None, shift=0):
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0[lo:hi].clone(), xmc.E4M3), num_chunks=k,
                           num_labels_global=glob or L, label_offset=lo if off is None else off)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding="stochastic", sr_impl="philox")
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li - shift), cfg, xmc.RoundingRng(11), 0)
    torch.cuda.synchronize()
    return gx

half = L // 2
gx1 = run(0, L)
gxa = run(0, half)
gxb = run(half, L)
d = (gxa + gxb - gx1).abs()
print("max diff", float(d.max()), "bad frac", float((d > 1e-3).float().mean()))
bad = (d > 1e-3)
print("bad rows(samples)", bad.any(1).nonzero().flatten()[:20].tolist())
print("bad cols", bad.any(0).nonzero().flatten()[:40].tolist(), int(bad.any(0).sum()))
# shard b as a standalone head with shifted labels
keep = (li >= half)
gxb2 = run(half, L, off=0, glob=L - half, shift=half)
print("b vs standalone", float((gxb - gxb2).abs().max()))
gxa2 = run(0, half, off=0, glob=half)
print("a vs standalone", float((gxa - gxa2).abs().max()))
