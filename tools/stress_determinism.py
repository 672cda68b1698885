"""Determinism stress: the same head step repeated (and with a different chunk
count) must give bit-identical W.  Run on the GPU box; prints mismatch counts."""
import sys, os, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11168_b200 as xmc
from oracle import lpxmc_oracle as O

def run(L, lo, hi, B, fname, k, precision, impl, W0, X, si, li):
    fmt = xmc.parse_format(fname)
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0.clone(), fmt), num_chunks=k, num_labels_global=L,
                           label_offset=lo, precision=precision)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic", sr_impl=impl)
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(21), 3)
    return head.weights.values.view(torch.uint8).clone(), gx

cases = [(8_623_847, 8, 5, 128, "e4m3"), (8_623_847, 8, 0, 128, "e4m3"), (2_812_281, 1, 0, 256, "e4m3"),
         (670_091, 1, 0, 256, "e4m3"), (131_073, 1, 0, 512, "bf16")]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for (L, world, rank, B, fname) in cases:
    lo, hi = xmc.partition(L, world)[rank]
    fmt = xmc.parse_format(fname)
    g = torch.Generator(device="cuda"); g.manual_seed(17)
    W0 = torch.empty((hi - lo, 768), dtype=fmt.torch_dtype, device="cuda")
    for r0 in range(0, hi - lo, 262_144):
        r1 = min(hi - lo, r0 + 262_144)
        W0[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, 768), generator=g, device="cuda") * 0.02, fmt)
    rs = np.random.default_rng(8)
    X = rs.normal(size=(B, 768)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, 9.0, seed=9)
    for precision in ("operand", "reference"):
        base, gx0 = run(L, lo, hi, B, fname, 2, precision, "hash", W0, X, si, li)
        bad_same, bad_k = 0, 0
        t0 = time.time()
        for r in range(reps):
            w, gx = run(L, lo, hi, B, fname, 2 if r % 2 == 0 else 1, precision, "hash", W0, X, si, li)
            n = int((w != base).sum())
            if n:
                if r % 2 == 0: bad_same += 1
                else: bad_k += 1
                rows = torch.nonzero((w != base).any(dim=1)).flatten()
                print(f"  rep {r} k={2 if r % 2 == 0 else 1}: {n} bytes differ in {rows.numel()} rows, "
                      f"first rows {rows[:8].tolist()}", flush=True)
        print(f"L={L} shard {rank}/{world} B={B} {fname} {precision}: {reps} reps, same-k mismatches {bad_same}, "
              f"k=1 mismatches {bad_k} ({time.time() - t0:.1f}s)", flush=True)
