"""Per-kernel timing of the head kernels in isolation (one C4 chunk by default):
forward (logits+G), backward in three modes (update only, grad_X only, both).
Device times come from the library's CUDA-event profiler.

    python tools/bench_kernels.py [--rows 351536] [--batch 256] [--fmt e4m3] [--iters 10]
"""

import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11168_b200 as xmc  # noqa: E402
from paper_2510_11168_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=351_536)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--fmt", default="e4m3")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounding", default="stochastic")
    a = ap.parse_args()
    fmt = xmc.parse_format(a.fmt)
    L, B, D = a.rows, a.batch, a.dim
    W = xmc.cast_native(torch.randn(L, D, device="cuda") * 0.02, fmt)
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, fmt), num_chunks=1)
    X = torch.randn(B, D, device="cuda")
    G = torch.rand(L, B, device="cuda") * 0.5
    acc = torch.zeros(B, D, device="cuda")
    cfg = xmc.SgdSrConfig(lr=1e-3, weight_decay=1e-4, fmt=fmt, rounding=a.rounding)
    args = _lib.StepArgs(cfg.lr, cfg.weight_decay, cfg.rounding_code, 0, 0, 1, xmc.HEAD_WEIGHTS_TAG)
    h = head.handle(B, 1024)
    lib = _lib.load()
    si = torch.zeros(1, dtype=torch.int32, device="cuda")
    li = torch.zeros(1, dtype=torch.int32, device="cuda")
    gx = torch.empty(B, D, device="cuda")
    res = {}

    def run(name, fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        _lib.profile_read()
        _lib.profile_enable(True)
        for _ in range(a.iters):
            fn()
        torch.cuda.synchronize()
        _lib.profile_enable(False)
        mf, nf, mb, nb = _lib.profile_read()
        res[name] = {"fwd_ms": mf / max(nf, 1), "bwd_ms": mb / max(nb, 1), "n_fwd": nf / a.iters,
                     "n_bwd": nb / a.iters}

    st = _lib.stream_ptr
    run("bwd_update_only", lambda: _lib.check(lib.xmc_head_backward(
        h.h, W.data_ptr(), G.data_ptr(), B, X.data_ptr(), B, 0, L, None, 0, 1, ctypes.byref(args), st())))
    run("bwd_gx_only", lambda: _lib.check(lib.xmc_head_backward(
        h.h, W.data_ptr(), G.data_ptr(), B, None, B, 0, L, acc.data_ptr(), 1, 0, None, st())))
    run("bwd_both", lambda: _lib.check(lib.xmc_head_backward(
        h.h, W.data_ptr(), G.data_ptr(), B, X.data_ptr(), B, 0, L, acc.data_ptr(), 1, 1, ctypes.byref(args),
        st())))
    run("step_1chunk", lambda: _lib.check(lib.xmc_head_step(
        h.h, W.data_ptr(), X.data_ptr(), B, si.data_ptr(), li.data_ptr(), 1, ctypes.byref(args),
        gx.data_ptr(), None, st())))
    eb = 1 if a.fmt == "e4m3" else 2
    for k, v in res.items():
        ms = v["bwd_ms"] if k.startswith("bwd") else v["fwd_ms"]
        mult = 4 if k == "bwd_both" else 2
        v["tflops"] = mult * B * L * D / (ms * 1e-3) / 1e12 if ms > 0 else None
    res["step_1chunk"]["fwd_tflops"] = 2 * B * L * D / (res["step_1chunk"]["fwd_ms"] * 1e-3) / 1e12
    print(json.dumps({"rows": L, "batch": B, "dim": D, "fmt": a.fmt, "results": res}, indent=1))


if __name__ == "__main__":
    main()
