import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2510_11168_b200 as xmc
from oracle import lpxmc_oracle as O
L, d, steps, lr, B, k, fname = 4096, 768, 5, 0.01, 256, 2, "bf16"
rs = np.random.default_rng(211)
fmt_o = O.parse_format(fname)
W = O.round_nearest(fmt_o, rs.normal(scale=0.02, size=(L, d)).astype(np.float32))
X = rs.normal(size=(B, d)).astype(np.float32)
si, li = O.synthetic_positives(L, B, 5.0, seed=212)
fmt = xmc.parse_format(fname)
head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, num_chunks=k)
oh = O.OracleHead(W.copy(), fmt_o, k)
cfg = xmc.SgdSrConfig(lr=lr, weight_decay=1e-4, fmt=fmt, rounding="nearest")
cfg_o = O.SgdSrConfig(lr=lr, weight_decay=1e-4, fmt=fmt_o, rounding="nearest")
for step in range(steps):
    xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(0), step)
    O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(0), step)
ref_scores = oh.scores(X)
gpu_scores = head.scores(torch.from_numpy(X)).cpu().numpy()
vals, labs = head.topk(torch.from_numpy(X), 5)
labs = labs.cpu().numpy(); vals = vals.cpu().numpy()
bad = 0
for s in range(B):
    tr = O.top_k_indices(ref_scores[s], 5); tg = O.top_k_indices(gpu_scores[s], 5)
    if not np.array_equal(labs[s], tg) or not np.array_equal(labs[s], tr):
        bad += 1
        if bad < 6:
            o = np.sort(ref_scores[s])[::-1]
            print(s, 'fused', labs[s], vals[s], '\n   gpu', tg, gpu_scores[s][tg], '\n   ref', tr, ref_scores[s][tr], 'margin', o[4]-o[5], 'maxdiff', np.abs(gpu_scores[s]-ref_scores[s]).max())
print('bad', bad)
