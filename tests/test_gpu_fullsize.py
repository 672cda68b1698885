"""Full-size (BASELINE C4: 2,812,281 labels x 768, batch 256, e4m3) parity
through size-independent properties:

* rows are independent in the update: a random subset of rows (plus rows
  with positives, chunk and tile edges, the last row) is recomputed by the
  oracle from the same W0 / X / positives / keys and must match the GPU
  within the stated bound (same bound as the small-size tests);
* chunk invariance at full size: k = 1 and k = 2 give bit-identical W and
  grad_X within fp32 tolerance;
* grad_X linearity: the full grad_X equals the sum of two label-sharded runs
  (the multi-GPU decomposition, here on one GPU).

These run the operand-precision mode (both modes for the invariances); the
reference-precision mode is checked against the unmodified reference at this
size in tests/test_gpu_reference.py.
"""

import os

import numpy as np
import pytest
import torch

from oracle import lpxmc_oracle as O

pytestmark = pytest.mark.gpu

L, D, B = 2_812_281, 768, 256


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11168_b200 as xmc
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    W0 = torch.empty((L, D), dtype=torch.float8_e4m3fn, device="cuda")
    for r0 in range(0, L, 262_144):
        r1 = min(L, r0 + 262_144)
        W0[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, D), generator=g, device="cuda") * 0.02, xmc.E4M3)
    rs = np.random.default_rng(3)
    X = rs.normal(size=(B, D)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, 36.17, seed=4)
    return xmc, W0, X, si, li


def _run(xmc, W0, X, si, li, k, rmode="stochastic", impl="splitmix64", lo=0, hi=L, precision="operand"):
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0[lo:hi].clone(), xmc.E4M3), num_chunks=k,
                           num_labels_global=L, label_offset=lo, precision=precision)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding=rmode, sr_impl=impl)
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(11), 0)
    return head, gx


def test_row_subset_matches_oracle(setup):
    xmc, W0, X, si, li = setup
    head, gx = _run(xmc, W0, X, si, li, k=2)
    rs = np.random.default_rng(5)
    rows = set(rs.choice(L, 400, replace=False).tolist())
    rows |= set(np.unique(li)[:100].tolist()) | set(np.unique(li)[-100:].tolist())
    half = L // 2
    rows |= {0, 127, 128, half - 1, half, half + 1, L - 129, L - 128, L - 1}
    rows = np.array(sorted(rows), dtype=np.int64)
    w0 = W0[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    Xq = O.round_nearest(O.E4M3, X)
    z = w0 @ Xq.T                                                      # (R, B)
    pos = np.zeros_like(z, dtype=bool)
    idx = {r: i for i, r in enumerate(rows)}
    for s, l in zip(si, li):
        if int(l) in idx:
            pos[idx[int(l)], s] = True
    G = np.clip(1.0 / (1.0 + np.exp(-z)), O.SIG_LO, O.SIG_HI).astype(np.float32) - pos.astype(np.float32)
    Gq = O.quantize_g_operand(G, O.E4M3)
    cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=O.E4M3, rounding="stochastic")
    gidx = rows[:, None].astype(np.uint64) * np.uint64(D) + np.arange(D, dtype=np.uint64)[None, :]
    ref = O.sgd_sr_values(w0, Gq @ Xq, cfg, O.RoundingRng(11), 0, O.HEAD_WEIGHTS_TAG, gidx)
    got = head.weights.values[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    same = np.mean(got.view(np.uint32) == ref.view(np.uint32))
    assert same > 0.99, same
    # bound: one grid ulp + lr * (accumulation noise + 2 operand-grid flips of G)
    Xa = np.abs(Xq.astype(np.float64))
    err = 2.0 ** -17 * (np.abs(Gq) @ Xa)
    uG = O._ulp_of(O.E5M2, np.abs(Gq) * 256.0) / 256.0
    err += 2 * (uG[:, :, None] * Xa[None]).max(axis=1)
    ulp = O._ulp_of(O.E4M3, np.maximum(np.abs(got), np.abs(ref)).astype(np.float64))
    assert np.all(np.abs(got.astype(np.float64) - ref) <= ulp + 0.05 * err * 1.01 + 1e-30)
    assert torch.isfinite(gx).all()


@pytest.mark.parametrize("precision", ["operand", "reference"])
def test_chunk_invariance_and_shard_linearity(setup, precision):
    xmc, W0, X, si, li = setup
    h1, gx1 = _run(xmc, W0, X, si, li, k=1, rmode="stochastic", impl="hash", precision=precision)
    h2, gx2 = _run(xmc, W0, X, si, li, k=2, rmode="stochastic", impl="hash", precision=precision)
    assert torch.equal(h1.weights.values.view(torch.uint8), h2.weights.values.view(torch.uint8))
    # grad_X: the chunking changes the fp32 summation order of 2.8M label
    # contributions (TMEM windows of 32 tiles, then the partial slots); in
    # reference precision every contribution is the sum of three exact plane
    # products, so values that cancel to near zero keep a few ulps of max|grad_X|
    atol = 1e-4 if precision == "operand" else max(1e-4, 2e-6 * float(gx1.abs().max()))
    torch.testing.assert_close(gx1, gx2, rtol=1e-5, atol=atol)
    del h2
    half = L // 2
    ha, gxa = _run(xmc, W0, X, si, li, k=1, impl="hash", lo=0, hi=half, precision=precision)
    hb, gxb = _run(xmc, W0, X, si, li, k=1, impl="hash", lo=half, hi=L, precision=precision)
    torch.testing.assert_close(gxa + gxb, gx1, rtol=1e-5, atol=atol)
    # global-row RNG keys: shard weights equal the single-GPU rows bit for bit
    assert torch.equal(ha.weights.values.view(torch.uint8), h1.weights.values[:half].view(torch.uint8))
    assert torch.equal(hb.weights.values.view(torch.uint8), h1.weights.values[half:].view(torch.uint8))


def test_fused_topk_full_size(setup):
    """Streaming top-k over all 2.8M labels equals the ranking of the same
    logits materialised slab by slab (merge with ties toward the lower label)."""
    xmc, W0, X, si, li = setup
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0, xmc.E4M3))
    Xt = torch.from_numpy(X).cuda()
    vals, labs = head.topk(Xt, 5)
    cand_v, cand_l = [], []
    for r0 in range(0, L, 400_000):
        r1 = min(L, r0 + 400_000)
        sc = xmc.ChunkedHead(xmc.QuantizedMatrix(W0[r0:r1], xmc.E4M3)).scores(Xt)
        order = torch.sort(-sc, dim=1, stable=True).indices[:, :5]
        cand_v.append(torch.gather(sc, 1, order))
        cand_l.append(order + r0)
    from paper_2510_11168_b200.parallel import merge_topk
    ref = merge_topk(torch.cat(cand_v, 1), torch.cat(cand_l, 1), 5)
    assert torch.equal(labs, ref)


def test_more_label_tiles_than_shared_memory_counters():
    """A rank with more than 48k label tiles (> 6.3M labels; the bucketing
    scan then runs from global memory) and more than 12k positives (the
    multi-CTA bucketing path): rows [hi - 100k, hi) must equal, bit for bit,
    the same rows updated by a small shard (single-CTA bucketing), and the
    positives near the end of the label range must be applied."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11168_b200 as xmc
    Lb, lo_s = 6_500_000, 6_400_000
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    W0 = torch.empty((Lb, D), dtype=torch.float8_e4m3fn, device="cuda")
    for r0 in range(0, Lb, 524_288):
        r1 = min(Lb, r0 + 524_288)
        W0[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, D), generator=g, device="cuda") * 0.02, xmc.E4M3)
    rs = np.random.default_rng(13)
    X = rs.normal(size=(B, D)).astype(np.float32)
    si, li = O.synthetic_positives(Lb, B, 60.0, seed=14)
    # plus 40 positives per sample inside the compared shard
    si2 = np.repeat(np.arange(B, dtype=np.int64), 40)
    li2 = rs.integers(lo_s, Lb, size=si2.size)
    si, li = np.concatenate([si, si2]), np.concatenate([li, li2])
    assert si.size > 12_288
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding="stochastic", sr_impl="splitmix64")
    full = xmc.ChunkedHead(xmc.QuantizedMatrix(W0.clone(), xmc.E4M3), num_chunks=5)
    xmc.head_update(full, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(11), 0)
    # the shard run sees the same global labels (out-of-shard ones are skipped)
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0[lo_s:].clone(), xmc.E4M3), num_chunks=1,
                           num_labels_global=Lb, label_offset=lo_s)
    xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(11), 0)
    a = full.weights.values[lo_s:].view(torch.uint8)
    b_ = head.weights.values.view(torch.uint8)
    assert torch.equal(a, b_), f"{int((a != b_).sum())} bytes differ"
    # the positives moved their rows (sigma - 1 < 0 pushes W up along X)
    assert not torch.equal(a, W0[lo_s:].view(torch.uint8))
