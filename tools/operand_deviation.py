"""Deviation of the operand-precision mode (the bench's production path) from
the unmodified reference, modelled with the oracle (the GPU matches this
model to > 99 % bitwise, tests/test_gpu_parity.py): one head step on the same
W0 / X / positives / keys, G rounded to the backward operand (e5m2(2^8 g) or
e4m3(2^8 g) for an e4m3 head, bf16(g) for a bf16 head) vs the reference's
fp32 G.  Prints the fraction of bit-identical weights, the grid-ulp histogram
and the relative grad_X error.  Test infrastructure (runs on the CPU).

    python tools/operand_deviation.py [--labels 4096] [--dim 768] [--batch 256]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lpxmc_oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--labels", type=int, default=4096)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--batch", type=int, default=256)
    a = ap.parse_args()
    out = []
    for fname, gq, rmode in (("e4m3", "bf16", "nearest"), ("e4m3", "bf16", "stochastic"),
                             ("e4m3", "e5m2", "nearest"), ("e4m3", "e5m2", "stochastic"),
                             ("e4m3", "e4m3", "nearest"), ("bf16", True, "nearest"), ("bf16", True, "stochastic")):
        fmt = O.parse_format(fname)
        rs = np.random.default_rng(3)
        W0 = O.round_nearest(fmt, rs.normal(scale=0.02, size=(a.labels, a.dim)).astype(np.float32))
        X = rs.normal(size=(a.batch, a.dim)).astype(np.float32)
        si, li = O.synthetic_positives(a.labels, a.batch, 5.0, seed=4)
        cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding=rmode)
        res = {}
        for tag, g in (("ref", False), ("op", gq)):
            h = O.OracleHead(W0.copy(), fmt, 2)
            gx = O.head_update(h, X, si, li, cfg, O.RoundingRng(7), 0, g_quant=g)
            res[tag] = (h.values.copy(), gx)
        wr, wo = res["ref"][0], res["op"][0]
        u = np.abs(wr.astype(np.float64) - wo) / O._ulp_of(fmt, np.maximum(np.abs(wr), np.abs(wo)).astype(np.float64))
        u = np.rint(u).astype(np.int64)
        hist = {str(k): float(np.mean(u == k)) for k in range(0, 4)}
        hist[">=4"] = float(np.mean(u >= 4))
        gxe = float(np.abs(res["op"][1] - res["ref"][1]).max() / np.abs(res["ref"][1]).max())
        r = {"fmt": fname, "g_operand": gq if gq is not True else "bf16", "rounding": rmode,
             "bit_identical": float(np.mean(wr.view(np.uint32) == wo.view(np.uint32))),
             "ulp_hist": hist, "max_ulp": int(u.max()), "grad_x_max_rel_err": gxe}
        print(json.dumps(r), flush=True)
        out.append(r)


if __name__ == "__main__":
    main()
