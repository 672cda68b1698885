"""Time the fused streaming top-k (ChunkedHead.topk) at a BASELINE shape and
compare with materialised scores + torch.topk (slabbed).  CUDA events.

    python tools/bench_topk.py [--labels 2812281] [--batch 256] [--fmt e4m3] [--k 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11168_b200 as xmc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--labels", type=int, default=2_812_281)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--fmt", default="e4m3")
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    fmt = xmc.parse_format(a.fmt)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    W = torch.empty((a.labels, a.dim), dtype=fmt.torch_dtype, device="cuda")
    for r0 in range(0, a.labels, 262_144):
        r1 = min(a.labels, r0 + 262_144)
        W[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, a.dim), generator=g, device="cuda") * 0.02, fmt)
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, fmt))
    X = torch.randn((a.batch, a.dim), generator=g, device="cuda")
    for _ in range(3):
        v, l = head.topk(X, a.k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        v, l = head.topk(X, a.k)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    flops = 2.0 * a.labels * a.dim * a.batch
    # materialised reference ranking of the same logits, in label slabs
    slab = 262_144
    best_v = best_l = None
    sc = None
    e0.record()
    for r0 in range(0, a.labels, slab):
        r1 = min(a.labels, r0 + slab)
        sub = xmc.ChunkedHead(xmc.QuantizedMatrix(W[r0:r1], fmt))
        sc = sub.scores(X)
        tv, ti = torch.topk(sc, a.k, dim=1)
        ti = ti + r0
        if best_v is None:
            best_v, best_l = tv, ti
        else:
            cv, cl = torch.cat([best_v, tv], 1), torch.cat([best_l, ti], 1)
            o = torch.topk(cv, a.k, dim=1).indices
            best_v, best_l = torch.gather(cv, 1, o), torch.gather(cl, 1, o)
    e1.record()
    torch.cuda.synchronize()
    ms_mat = e0.elapsed_time(e1)
    agree = float((best_l == l).all(dim=1).float().mean())
    print(json.dumps({"labels": a.labels, "batch": a.batch, "fmt": a.fmt, "k": a.k, "ms_fused_topk": ms,
                      "tflops_fused": flops / (ms * 1e-3) / 1e12, "samples_per_s": a.batch / (ms * 1e-3),
                      "ms_materialised_slabs_torch_topk": ms_mat, "rows_agreeing": agree}))


if __name__ == "__main__":
    main()
