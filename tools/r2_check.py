"""Quick GPU check of the reference-precision mode against the reference's own
golden head steps (W1, gradX1) and of the operand mode against its oracle."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_11168_b200 as xmc
from oracle import lpxmc_oracle as O

G = np.load(os.path.join(ROOT, "tests", "golden", "lpxmc_golden.npz"))
n = int(G["head_ncases"])
for prec in ("reference",):
    for ci in range(n):
        p = f"head{ci}_"
        L, d, b, k = (int(v) for v in G[p + "meta"])
        lr, wd, drop, seed = G[p + "cfg"]
        fmt_name, rnd = str(G[p + "fmt"]), str(G[p + "rounding"])
        fmt = xmc.parse_format(fmt_name)
        head = xmc.ChunkedHead.from_float(torch.from_numpy(G[p + "W0"]), fmt, num_chunks=k, dropout_p=float(drop),
                                          precision=prec)
        cfg = xmc.SgdSrConfig(lr=float(lr), weight_decay=float(wd), fmt=fmt, rounding=rnd, sr_impl="splitmix64")
        gx = xmc.head_update(head, xmc.BatchInput(G[p + "X"], G[p + "sample_idx"], G[p + "label_idx"]), cfg,
                             xmc.RoundingRng(int(seed)), 0).cpu().numpy()
        W = head.weights.values.float().cpu().numpy()
        ofmt = O.parse_format(fmt_name)
        ref = G[p + "W1"]
        same = np.mean(W == ref)
        ulp = np.abs(W.astype(np.float64) - ref) / O._ulp_of(ofmt, np.maximum(np.abs(W), np.abs(ref)).astype(np.float64))
        gref = G[p + "gradX1"]
        rel = np.abs(gx - gref).max() / np.abs(gref).max()
        print(f"{prec:9s} case {ci} {fmt_name} {rnd:10s} k={k} drop={float(drop):.2f}: W same {same:.4f} "
              f"max ulp {ulp.max():.2f} >1ulp {np.mean(ulp > 1.0001):.4f} gradX maxrel {rel:.2e}")

# operand mode against the oracle with the same operand G
for gf in ("e5m2", "e4m3"):
    for ci in range(n):
        p = f"head{ci}_"
        L, d, b, k = (int(v) for v in G[p + "meta"])
        lr, wd, drop, seed = G[p + "cfg"]
        fmt_name, rnd = str(G[p + "fmt"]), str(G[p + "rounding"])
        if fmt_name != "e4m3" and gf == "e4m3":
            continue
        fmt = xmc.parse_format(fmt_name)
        head = xmc.ChunkedHead.from_float(torch.from_numpy(G[p + "W0"]), fmt, num_chunks=k, dropout_p=float(drop),
                                          precision="operand", g_format=gf)
        cfg = xmc.SgdSrConfig(lr=float(lr), weight_decay=float(wd), fmt=fmt, rounding=rnd, sr_impl="splitmix64")
        gx = xmc.head_update(head, xmc.BatchInput(G[p + "X"], G[p + "sample_idx"], G[p + "label_idx"]), cfg,
                             xmc.RoundingRng(int(seed)), 0).cpu().numpy()
        W = head.weights.values.float().cpu().numpy()
        ofmt = O.parse_format(fmt_name)
        oh = O.OracleHead(G[p + "W0"].copy(), ofmt, k, dropout_p=float(drop))
        gx_o = O.head_update(oh, G[p + "X"], G[p + "sample_idx"], G[p + "label_idx"],
                             O.SgdSrConfig(lr=float(lr), weight_decay=float(wd), fmt=ofmt, rounding=rnd),
                             O.RoundingRng(int(seed)), 0, g_quant=gf)
        print(f"operand/{gf} case {ci}: W same vs operand oracle {np.mean(W == oh.values):.4f} "
              f"vs reference W1 {np.mean(W == G[p + 'W1']):.4f}  gradX vs oracle maxrel "
              f"{np.abs(gx - gx_o).max() / np.abs(gx_o).max():.2e}")
