import time, sys, os, ctypes
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2510_11168_b200 as xmc
from paper_2510_11168_b200 import _lib
from oracle.lpxmc_oracle import synthetic_positives
L, D, B = 2812281, 768, 256
fmt = xmc.E4M3
W = torch.zeros((L, D), dtype=fmt.torch_dtype, device="cuda")
head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, fmt), num_chunks=2)
X = torch.randn((B, D), device="cuda")
si, li = synthetic_positives(L, B, 36.17, seed=1)
sid = torch.from_numpy(si.astype(np.int32)).cuda(); lid = torch.from_numpy(li.astype(np.int32)).cuda()
cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic")
rng = xmc.RoundingRng(0)
gx = torch.empty((B, D), device="cuda")
batch = xmc.BatchInput(X, sid, lid)
for s in range(5): xmc.head_update(head, batch, cfg, rng, s, check=False, grad_out=gx)
torch.cuda.synchronize()
# host-only cost of the python wrapper (GPU busy, async): enqueue time
t0 = time.perf_counter()
for s in range(50): xmc.head_update(head, batch, cfg, rng, s, check=False, grad_out=gx)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("enqueue us/step", (t1 - t0) / 50 * 1e6, "total ms/step", (t2 - t0) / 50 * 1e3)
# synchronous steps
t0 = time.perf_counter()
for s in range(50):
    xmc.head_update(head, batch, cfg, rng, s, check=False, grad_out=gx); torch.cuda.synchronize()
t1 = time.perf_counter()
print("sync ms/step", (t1 - t0) / 50 * 1e3)
# raw C call
h = head.handle(B, len(si))
args = xmc.head._step_args(cfg, rng, 0, head.tensor_id)
lib = _lib.load(); st = _lib.stream_ptr()
t0 = time.perf_counter()
for s in range(50):
    lib.xmc_head_step_kahan(h.h, W.data_ptr(), None, X.data_ptr(), B, sid.data_ptr(), lid.data_ptr(), sid.numel(), ctypes.byref(args), gx.data_ptr(), None, st)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("raw C enqueue us/step", (t1 - t0) / 50 * 1e6)
