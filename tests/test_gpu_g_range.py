"""Range of the operand-precision G of an e4m3 head in a trained-head regime
(logits ~ N(-9 ... -12, 2): the sigmoid of most labels far below 2^-8).

The reference clips the sigmoid at 2^-24 (head.py:47-48) and uses fp32 G.
The default operand format e5m2(2^8 g) represents that whole range (its
smallest subnormal 2^-16 is exactly 2^8 * 2^-24); e4m3(2^8 g) flushes every
sigmoid below ~2^-18 to zero.  Readout: W gets a column of ones and X a zero
in that column, so grad_X[:, 1] = sum_l Gq[l, b] -- the sum of the G operand
the backward GEMMs actually used, per sample.  Criterion: the relative error
of that sum against the fp32 sum of the reference's G is <= 1e-2, and (on the
bit-identical oracle restatement of the operand rounding) fewer than 1 % of
the entries flush to zero."""

import numpy as np
import pytest
import torch

from oracle import lpxmc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xmc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11168_b200 as xmc
    return xmc


def _problem(shift, L=65536, d=128, B=128, seed=0):
    rs = np.random.default_rng(seed)
    W = np.zeros((L, d), np.float32)
    W[:, 0] = shift                                   # bias feature: logits centred at `shift`
    W[:, 1] = 1.0                                     # readout column: grad_X[:, 1] = sum_l G[l, :]
    W[:, 2:] = rs.normal(scale=2.0 / np.sqrt(d - 2), size=(L, d - 2))
    W = O.round_nearest(O.E4M3, W)
    X = rs.normal(size=(B, d)).astype(np.float32)
    X[:, 0] = 1.0
    X[:, 1] = 0.0
    return W, X


@pytest.mark.parametrize("shift", [-9.0, -10.0, -12.0])
def test_e5m2_operand_keeps_trained_regime_gradient(xmc, shift):
    W, X = _problem(shift)
    L, B = W.shape[0], X.shape[0]
    Xq = O.round_nearest(O.E4M3, X)
    z = W @ Xq.T
    assert abs(float(np.median(z)) - shift) < 0.5 and 1.5 < float(np.std(z)) < 2.5
    G = O.logit_gradient(z, np.zeros(0, np.int64), np.zeros(0, np.int64), (0, L))
    sums = {}
    for gf in ("e5m2", "e4m3"):
        head = xmc.ChunkedHead.from_float(torch.from_numpy(W), xmc.E4M3, precision="operand", g_format=gf)
        cfg = xmc.SgdSrConfig(lr=1e-3, fmt=xmc.E4M3, rounding="nearest")
        gx = xmc.head_update(head, xmc.BatchInput(X, np.zeros(0), np.zeros(0)), cfg, xmc.RoundingRng(0), 0)
        sums[gf] = gx[:, 1].double().cpu().numpy()
        Gq = O.quantize_g_operand(G, O.E4M3, gf)
        # the GPU used exactly this operand (bit-identical rounding, tested in
        # test_gpu_parity.py): its per-sample sums agree to fp32 accumulation
        np.testing.assert_allclose(sums[gf], Gq.astype(np.float64).sum(axis=0), rtol=1e-4)
        if gf == "e5m2":
            assert float(np.mean(Gq == 0)) < 0.01
    ref = G.astype(np.float64).sum(axis=0)
    rel = np.abs(sums["e5m2"] - ref) / ref
    assert rel.max() <= 1e-2, rel.max()
    # the reference-precision mode has no operand rounding at all
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), xmc.E4M3)
    gx = xmc.head_update(head, xmc.BatchInput(X, np.zeros(0), np.zeros(0)),
                         xmc.SgdSrConfig(lr=1e-3, fmt=xmc.E4M3, rounding="nearest"), xmc.RoundingRng(0), 0)
    rel_ref = np.abs(gx[:, 1].double().cpu().numpy() - ref) / ref
    assert rel_ref.max() <= 1e-4, rel_ref.max()
    print(f"shift {shift}: max rel. error of sum G -- e5m2 {rel.max():.2e}, "
          f"e4m3 {(np.abs(sums['e4m3'] - ref) / ref).max():.2e}, reference precision {rel_ref.max():.2e}; "
          f"e4m3 flushed {np.mean(O.quantize_g_operand(G, O.E4M3, 'e4m3') == 0):.3f}")
