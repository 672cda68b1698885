"""Host-side cost of one head_update call vs its device time (measurement
tool): if the CPU enqueue time per step exceeds the device time, the GPU
idles between steps and ms/step measures Python, not kernels."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_11168_b200 as xmc  # noqa: E402
from oracle.lpxmc_oracle import synthetic_positives  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 351_536
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
D, B = 768, 256
dev = torch.device("cuda")
W = xmc.cast_native(torch.randn((L, D), device=dev) * 0.02, xmc.E4M3)
head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, xmc.E4M3), num_chunks=k, num_labels_global=L)
si, li = synthetic_positives(L, B, 5.45, seed=1)
X = torch.randn((B, D), device=dev)
batch = xmc.BatchInput(X, torch.from_numpy(si.astype(np.int32)).to(dev), torch.from_numpy(li.astype(np.int32)).to(dev))
cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding="stochastic", sr_impl="philox")
rng = xmc.RoundingRng(0)
gx = torch.empty((B, D), device=dev)
for s in range(10):
    xmc.head_update(head, batch, cfg, rng, s, check=False, grad_out=gx)
torch.cuda.synchronize()
n = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for s in range(n):
    xmc.head_update(head, batch, cfg, rng, 10 + s, check=False, grad_out=gx)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
print(f"L={L} k={k}: host {1e3 * (t1 - t0) / n:.4f} ms/call, device {e0.elapsed_time(e1) / n:.4f} ms/step")
# device time with the queue pre-filled: enqueue behind a long sleep kernel
torch.cuda._sleep(int(2e9))
e0.record()
for s in range(n):
    xmc.head_update(head, batch, cfg, rng, 10 + s, check=False, grad_out=gx)
e1.record()
torch.cuda.synchronize()
print(f"  queue pre-filled: device {e0.elapsed_time(e1) / n:.4f} ms/step")
