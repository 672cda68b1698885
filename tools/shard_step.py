"""Device time of one rank's step in an N-way label-sharded run, on one GPU
(measurement tool): rank 0's shard of L_global labels, the GLOBAL positive
list (mean labels/sample as in bench.py), k chunks.  Prints ms/step and the
library's fwd / bwd kernel ms, i.e. what the N-GPU scaling run costs per
rank before the grad_X all-reduce.

    python tools/shard_step.py [world=8] [mean_labels=36.17] [chunks=1]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11168_b200 as xmc  # noqa: E402
from paper_2510_11168_b200 import _lib  # noqa: E402
from oracle.lpxmc_oracle import synthetic_positives  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mean = float(sys.argv[2]) if len(sys.argv) > 2 else 36.17
k = int(sys.argv[3]) if len(sys.argv) > 3 else 1
L, D, B = 2_812_281, 768, 256
lo, hi = xmc.partition(L, world)[0]
dev = torch.device("cuda")
W = xmc.cast_native(torch.randn((hi - lo, D), device=dev) * 0.02, xmc.E4M3)
head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, xmc.E4M3), num_chunks=k, num_labels_global=L, label_offset=lo,
                       precision="operand")
si, li = synthetic_positives(L, B, mean, seed=1)
X = torch.randn((B, D), device=dev)
batch = xmc.BatchInput(X, torch.from_numpy(si.astype(np.int32)).to(dev), torch.from_numpy(li.astype(np.int32)).to(dev))
cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding="stochastic")
rng = xmc.RoundingRng(0)
gx = torch.empty((B, D), device=dev)
for s in range(10):
    xmc.head_update(head, batch, cfg, rng, s, check=False, grad_out=gx)
torch.cuda.synchronize()
n = 200
_lib.profile_read()
_lib.profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for s in range(n):
    xmc.head_update(head, batch, cfg, rng, 10 + s, check=False, grad_out=gx)
e1.record()
torch.cuda.synchronize()
_lib.profile_enable(False)
mf, nf, mb, nb = _lib.profile_read()
print(f"world={world} shard={hi - lo} nnz={len(si)} k={k}: {e0.elapsed_time(e1) / n:.4f} ms/step "
      f"(fwd {mf / n:.4f}, bwd {mb / n:.4f})")
