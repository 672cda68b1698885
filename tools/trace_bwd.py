"""Pipeline timeline of the first backward CTA (measurement only).

    XMC_TRACE=1 python tools/trace_bwd.py [--rows 351536] [--mode both|update|gx]

Events per tile (clock64): 0 producer W issued, 1 producer G issued, 2 MMA saw
W, 3 MMA saw the last G slot, 4 MMA issued everything, 5 epilogue saw W,
6 epilogue saw dW (t_full), 7 epilogue stored W_new.
"""

import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("XMC_TRACE", "1")
import paper_2510_11168_b200 as xmc  # noqa: E402
from paper_2510_11168_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=351_536)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--mode", default="both")
    a = ap.parse_args()
    L, B, D = a.rows, a.batch, 768
    fmt = xmc.E4M3
    W = xmc.cast_native(torch.randn(L, D, device="cuda") * 0.02, fmt)
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, fmt), num_chunks=1)
    X = torch.randn(B, D, device="cuda")
    G = torch.rand(L, B, device="cuda") * 0.5
    acc = torch.zeros(B, D, device="cuda")
    cfg = xmc.SgdSrConfig(lr=1e-3, weight_decay=1e-4, fmt=fmt, rounding="stochastic")
    args = _lib.StepArgs(cfg.lr, cfg.weight_decay, cfg.rounding_code, 0, 0, 1, xmc.HEAD_WEIGHTS_TAG)
    h = head.handle(B, 1024)
    lib = _lib.load()
    lib.xmc_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    st = _lib.stream_ptr
    upd, gx = {"both": (1, 1), "update": (1, 0), "gx": (0, 1)}[a.mode]
    for _ in range(4):
        _lib.check(lib.xmc_head_backward(h.h, W.data_ptr(), G.data_ptr(), B, X.data_ptr(), B, 0, L,
                                         acc.data_ptr() if gx else None, gx, upd,
                                         ctypes.byref(args) if upd else None, st()))
    torch.cuda.synchronize()
    buf = np.zeros((512, 16), dtype=np.uint64)
    _lib.check(lib.xmc_trace_read(buf.ctypes.data, buf.size))
    n = int((buf[:, 7] > 0).sum()) if upd else int((buf[:, 4] > 0).sum())
    t = buf[:n].astype(np.int64)
    t -= t[0, 0]
    lo, hi = 5, n - 2
    d = lambda a_, b_: np.median(t[lo:hi, b_] - t[lo:hi, a_])  # noqa: E731
    per = np.median(np.diff(t[lo:hi, 4]))
    print(f"tiles traced {n}; median cycles per tile (MMA issue-to-issue) {per:.0f}")
    print(f"  W latency  (issue->MMA saw)   {d(0, 2):7.0f}")
    print(f"  G latency  (issue->MMA saw)   {d(1, 3):7.0f}")
    print(f"  MMA w->lastG wait             {d(2, 3):7.0f}")
    print(f"  MMA issue span                {d(3, 4):7.0f}")
    print(f"    MMA: W seen -> t_empty      {d(2, 8):7.0f}")
    print(f"    MMA: t_empty -> G kc0 seen  {d(8, 9):7.0f}")
    print(f"    MMA: kc0 dW MMAs issued     {d(9, 10):7.0f}")
    print(f"    MMA: -> G kc1 seen          {d(10, 3):7.0f}")
    if upd:
        print(f"  epi: W seen -> dW seen        {d(5, 6):7.0f}")
        print(f"  epi: dW seen -> stored        {d(6, 7):7.0f}")
        print(f"  epi period (stored->stored)   {np.median(np.diff(t[lo:hi, 7])):7.0f}")
        print(f"  MMA issued -> epi saw dW      {d(4, 6):7.0f}")
    print(f"  producer W issue lead over MMA {d(0, 4):7.0f}")
    np.set_printoptions(linewidth=200)
    print("rows 8..16 (relative cycles):")
    print((t[8:16] - t[8, 0])[:, :11])


if __name__ == "__main__":
    main()
