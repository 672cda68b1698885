"""Parity at the other BASELINE.json configurations (C1 is the CPU golden case,
C4 is tests/test_gpu_fullsize.py):

* C2  LF-AmazonTitles-131K shape: 131,073 labels, d=768, batch 512, bf16, 1 chunk;
* C3  Amazon-670K shape: 670,091 labels, batch 256, e4m3, 4 chunks;
* C5  LF-Paper2Keywords-8.6M shape, one rank's label shard of an 8-way split
      (rank 0 and rank 5), batch 128 as in the paper, e4m3.

Each runs one full head step and checks, through size-independent
properties: a row subset (random rows, rows with positives, chunk / tile /
shard edges) against the oracle recomputed from the same W0, X, positives
and global-row keys -- the UNMODIFIED oracle in the default
reference-precision mode (parity_util bound), the oracle on the same operand
G in the operand mode; grad_X of the reference-precision step against an
fp32 restatement over every label of the shard (rtol 1e-4); chunk invariance
(bitwise W) and grad_X within fp32 tolerance; finite outputs.
"""

import numpy as np
import pytest
import torch

from oracle import lpxmc_oracle as O
from parity_util import reference_weight_report, torch_fp32_grad_x

pytestmark = pytest.mark.gpu

CONFIGS = {
    # name: (L_global, batch, fmt, chunks, shard (world, rank) or None, mean labels/sample)
    "C2": (131_073, 512, "bf16", 1, None, 5.15),
    "C3": (670_091, 256, "e4m3", 4, None, 5.45),
    "C5r0": (8_623_847, 128, "e4m3", 2, (8, 0), 9.03),
    "C5r5": (8_623_847, 128, "e4m3", 2, (8, 5), 9.03),
}
D = 768


def _setup(xmc, name):
    L, B, fname, k, shard, mean = CONFIGS[name]
    fmt = xmc.parse_format(fname)
    lo, hi = (0, L) if shard is None else xmc.partition(L, shard[0])[shard[1]]
    g = torch.Generator(device="cuda")
    g.manual_seed(17)
    W0 = torch.empty((hi - lo, D), dtype=fmt.torch_dtype, device="cuda")
    for r0 in range(0, hi - lo, 262_144):
        r1 = min(hi - lo, r0 + 262_144)
        W0[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, D), generator=g, device="cuda") * 0.02, fmt)
    rs = np.random.default_rng(8)
    X = rs.normal(size=(B, D)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, mean, seed=9)
    return L, B, fmt, k, lo, hi, W0, X, si, li


def _step(xmc, fmt, W0, X, si, li, L, lo, k, impl, precision="operand"):
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0.clone(), fmt), num_chunks=k, num_labels_global=L,
                           label_offset=lo, precision=precision)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic", sr_impl=impl)
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(21), 3)
    return head, gx


@pytest.mark.parametrize("precision", ["reference", "operand"])
@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_row_subset_matches_oracle(name, precision):
    import paper_2510_11168_b200 as xmc
    L, B, fmt, k, lo, hi, W0, X, si, li = _setup(xmc, name)
    head, gx = _step(xmc, fmt, W0, X, si, li, L, lo, k, "splitmix64", precision)
    assert torch.isfinite(gx).all()
    n = hi - lo
    rs = np.random.default_rng(6)
    rows = set(rs.choice(n, min(n, 300), replace=False).tolist())
    local_pos = np.unique(li[(li >= lo) & (li < hi)]) - lo
    rows |= set(local_pos[:150].tolist()) | set(local_pos[-50:].tolist())
    for c0, c1 in xmc.partition(n, k):
        rows |= {c0, min(c0 + 127, n - 1), min(c0 + 128, n - 1), c1 - 1}
    rows = np.array(sorted(rows), dtype=np.int64)
    of = O.parse_format(fmt.name)
    w0 = W0[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    Xq = O.round_nearest(of, X)
    z = w0 @ Xq.T
    pos = np.zeros_like(z, dtype=bool)
    idx = {int(r) + lo: i for i, r in enumerate(rows)}
    for s, l in zip(si, li):
        if int(l) in idx:
            pos[idx[int(l)], s] = True
    G = np.clip(1.0 / (1.0 + np.exp(-z)), O.SIG_LO, O.SIG_HI).astype(np.float32) - pos.astype(np.float32)
    cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=of, rounding="stochastic")
    gidx = (rows[:, None] + lo).astype(np.uint64) * np.uint64(D) + np.arange(D, dtype=np.uint64)[None, :]
    got = head.weights.values[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    if precision == "reference":
        ref = O.sgd_sr_values(w0, G @ Xq, cfg, O.RoundingRng(21), 3, O.HEAD_WEIGHTS_TAG, gidx)
        same, over1, ok = reference_weight_report(got, ref, of, 0.05, G, Xq, sr=True)
        assert same >= 0.999 and ok, (same, over1)
        gx_ref = torch_fp32_grad_x(W0, Xq, si, li, label0=lo).cpu().numpy()
        err = np.abs(gx.cpu().numpy() - gx_ref).max() / np.abs(gx_ref).max()
        assert err <= 1e-4, err
        return
    Gq = O.quantize_g_operand(G, of)
    ref = O.sgd_sr_values(w0, Gq @ Xq, cfg, O.RoundingRng(21), 3, O.HEAD_WEIGHTS_TAG, gidx)
    same = np.mean(got.view(np.uint32) == ref.view(np.uint32))
    assert same > 0.99, same
    # bound: one grid ulp + lr * (fp32 accumulation noise + 2 operand-grid flips of G)
    Xa = np.abs(Xq.astype(np.float64))
    err = 2.0 ** -17 * (np.abs(Gq) @ Xa)
    if of.name == "e4m3":
        uG = O._ulp_of(O.E5M2, np.abs(Gq) * 256.0) / 256.0
    else:
        uG = O._ulp_of(O.BF16, np.abs(Gq).astype(np.float64))
    err += 2 * (uG[:, :, None] * Xa[None]).max(axis=1)
    ulp = O._ulp_of(of, np.maximum(np.abs(got), np.abs(ref)).astype(np.float64))
    assert np.all(np.abs(got.astype(np.float64) - ref) <= ulp + 0.05 * err * 1.01 + 1e-30)


@pytest.mark.parametrize("name", ["C2", "C3", "C5r5"])
def test_config_chunk_invariance(name):
    import paper_2510_11168_b200 as xmc
    L, B, fmt, k, lo, hi, W0, X, si, li = _setup(xmc, name)
    k2 = 3 if k == 1 else 1
    ha, gxa = _step(xmc, fmt, W0, X, si, li, L, lo, k, "hash")
    hb, gxb = _step(xmc, fmt, W0, X, si, li, L, lo, k2, "hash")
    assert torch.equal(ha.weights.values.view(torch.uint8), hb.weights.values.view(torch.uint8))
    torch.testing.assert_close(gxa, gxb, rtol=1e-5, atol=1e-4)
