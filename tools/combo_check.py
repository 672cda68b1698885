"""Robustness sweep (GPU): every precision / G format / optimizer / Kahan /
dropout / batch combination runs two head steps at a small size without
error, with finite grad_X and weights.  Prints one line per combination."""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_11168_b200 as xmc  # noqa: E402
from oracle import lpxmc_oracle as O  # noqa: E402

L, d = 3000, 256
bad = 0
for fmt_name, prec, gfmt, kahan, drop, B, rounding in itertools.product(
        ["e4m3", "bf16"], ["operand", "reference"], ["e5m2", "e4m3", "bf16"], [None, "bf16", "fp32"],
        [0.0, 0.2], [100, 256, 512, 1500], ["stochastic", "nearest"]):
    if fmt_name == "bf16" and gfmt != "e5m2":
        continue   # a bf16 head's G is always bf16
    if prec == "reference" and gfmt != "e5m2":
        continue   # g_format applies to the operand precision only
    tag = f"{fmt_name} {prec} g={gfmt} kahan={kahan} p={drop} B={B} {rounding}"
    try:
        rs = np.random.default_rng(1)
        f = xmc.parse_format(fmt_name)
        W = O.round_nearest(O.parse_format(fmt_name), rs.normal(scale=0.02, size=(L, d)).astype(np.float32))
        head = xmc.ChunkedHead.from_float(torch.from_numpy(W), f, num_chunks=2, precision=prec, g_format=gfmt,
                                          kahan=kahan, dropout_p=drop)
        X = rs.normal(size=(B, d)).astype(np.float32)
        si, li = O.synthetic_positives(L, B, 4.0, seed=2)
        cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=f, rounding=rounding, sr_impl="hash")
        for s in range(2):
            gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(3), s)
        torch.cuda.synchronize()
        ok = bool(torch.isfinite(gx).all()) and bool(torch.isfinite(head.weights.values.float()).all())
        print("ok  " if ok else "BAD ", tag, flush=True)
        bad += 0 if ok else 1
    except NotImplementedError as e:
        print("n/a ", tag, "--", str(e)[:90], flush=True)
    except Exception as e:  # noqa: BLE001
        print("ERR ", tag, "--", type(e).__name__, str(e)[:120], flush=True)
        bad += 1
print("failures:", bad)
