"""Reference-precision mode (ChunkedHead(precision="reference"), the default)
against the UNMODIFIED reference: the golden head steps produced by lpxmc
itself (tests/golden/make_golden.py) and the oracle without any operand
quantisation of G.

The GPU forms the reference's fp32 G (head.py:181-196) and splits it exactly
into three bf16 planes, so both backward GEMMs multiply by the same fp32 G as
the reference (head.py:193-208, 236); W and X are exact in bf16.  What remains
is fp32 evaluation order (tensor-core vs OpenBLAS accumulation, CUDA vs numpy
expf).  Tolerances stated per test:
  * W: >= 99.9 % bit-identical after one step from the same W (>= 99.5 % on
    the 5-step trajectories); every element within one grid ulp (two with
    SR) plus the worst-case fp32 summation bound of its update value
    (parity_util.reference_weight_report);
  * grad_X: rtol 1e-4 (relative to max |grad_X|);
  * deterministic (RTN) training: per-step parity along the oracle's
    trajectory, and on independent 5-step runs P@1/3/5 equal and top-k label
    indices equal wherever the measured score difference cannot reorder them
    (north_star).
"""

import os

import numpy as np
import pytest
import torch

from oracle import lpxmc_oracle as O
from parity_util import fp32_update_noise, reference_weight_report, torch_fp32_grad_x

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "lpxmc_golden.npz"))
NCASES = int(GOLD["head_ncases"])


@pytest.fixture(scope="module")
def xmc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11168_b200 as xmc
    return xmc


def _rand_problem(L, d, B, fmt_name, seed, mean_labels=3.0, scale=0.02):
    rs = np.random.default_rng(seed)
    fmt = O.parse_format(fmt_name)
    W = O.round_nearest(fmt, rs.normal(scale=scale, size=(L, d)).astype(np.float32))
    X = rs.normal(size=(B, d)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, mean_labels, seed=seed + 1)
    return fmt, W, X, si, li


def _gx_close(got, ref, rtol=1e-4):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)
    assert err <= rtol, err


def _w_eff(W, p, seed, step):
    if p == 0.0:
        return W
    m = O.dropout_mask(O.RoundingRng(seed), step, p, (0, W.shape[0]), W.shape[1])
    return W * (m / np.float32(1.0 - p))


@pytest.mark.parametrize("ci", range(NCASES))
def test_head_update_matches_reference_golden(xmc, ci):
    """One full head step (bf16 / e4m3, RTN / splitmix64 SR, k = 1..4, keyed
    dropout) against lpxmc's own W1 and gradX1."""
    p = f"head{ci}_"
    L, d, b, k = (int(v) for v in GOLD[p + "meta"])
    lr, wd, drop, seed = (float(v) for v in GOLD[p + "cfg"])
    fname, rnd = str(GOLD[p + "fmt"]), str(GOLD[p + "rounding"])
    fmt, ofmt = xmc.parse_format(fname), O.parse_format(fname)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(GOLD[p + "W0"]), fmt, num_chunks=k, dropout_p=drop)
    assert head.precision == "reference"
    cfg = xmc.SgdSrConfig(lr=lr, weight_decay=wd, fmt=fmt, rounding=rnd, sr_impl="splitmix64")
    gx = xmc.head_update(head, xmc.BatchInput(GOLD[p + "X"], GOLD[p + "sample_idx"], GOLD[p + "label_idx"]), cfg,
                         xmc.RoundingRng(int(seed)), 0)
    _gx_close(gx.cpu().numpy(), GOLD[p + "gradX1"])
    Xq = O.round_nearest(ofmt, GOLD[p + "X"])
    W0 = GOLD[p + "W0"]
    G = O.logit_gradient(_w_eff(W0, drop, int(seed), 0) @ Xq.T, GOLD[p + "sample_idx"], GOLD[p + "label_idx"],
                         (0, L))
    same, over1, ok = reference_weight_report(head.weights.values.float().cpu().numpy(), GOLD[p + "W1"], ofmt, lr,
                                              G, Xq / np.float32(1.0 - drop), sr=rnd == "stochastic")
    assert same >= 0.999, same
    assert ok, (same, over1)


@pytest.mark.parametrize("fname,B,k", [("e4m3", 256, 2), ("bf16", 256, 2), ("bf16", 512, 1), ("e4m3", 100, 3),
                                       ("bf16", 48, 1)])
def test_rtn_training_trajectory_matches_oracle(xmc, fname, B, k):
    """Five RTN steps of a 4,096-label d = 768 head along the oracle's own
    trajectory (the GPU head is reset to the oracle's W before each step):
    every step's W >= 99.9 % bit-identical with the rest inside the fp32
    evaluation-order bound, grad_X at rtol 1e-4."""
    L, d, steps, lr = 4096, 768, 5, 0.01
    fmt_o, W, X, si, li = _rand_problem(L, d, B, fname, 201, mean_labels=5.0)
    fmt = xmc.parse_format(fname)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, num_chunks=k)
    oh = O.OracleHead(W.copy(), fmt_o, k)
    cfg = xmc.SgdSrConfig(lr=lr, weight_decay=1e-4, fmt=fmt, rounding="nearest")
    cfg_o = O.SgdSrConfig(lr=lr, weight_decay=1e-4, fmt=fmt_o, rounding="nearest")
    Xq = O.round_nearest(fmt_o, X)
    for step in range(steps):
        Wb = oh.values.copy()
        head.weights.values.copy_(xmc.cast_native(torch.from_numpy(Wb).cuda(), fmt))
        gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(0), step)
        gx_o = O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(0), step)
        _gx_close(gx.cpu().numpy(), gx_o)
        G = O.logit_gradient(Wb @ Xq.T, si, li, (0, L))
        same, over1, ok = reference_weight_report(head.weights.values.float().cpu().numpy(), oh.values, fmt_o, lr,
                                                  G, Xq)
        assert same >= 0.995 and ok, (step, same, over1)


@pytest.mark.parametrize("fname,B,k", [("e4m3", 256, 2), ("bf16", 256, 2), ("e4m3", 100, 3), ("bf16", 48, 1)])
def test_rtn_training_topk_and_p_at_k_equal_oracle(xmc, fname, B, k):
    """north_star's deterministic-mode target on two INDEPENDENT 5-step RTN
    runs (GPU vs unmodified oracle, no resync): P@1/3/5 (metrics.py:50-79) of
    the trained heads are equal, and every sample's top-5 label set
    (metrics.py:38-47; GPU: the fused streaming top-k) is equal to the
    oracle's except where the measured score differences of the two labels
    involved exceed their margin.  (Independent trajectories drift apart by
    the rare weight that an fp32 evaluation-order tie sent to the other grid
    neighbour; any other top-k difference would be a kernel error.)"""
    L, d, steps, lr = 4096, 768, 5, 0.01
    fmt_o, W, X, si, li = _rand_problem(L, d, B, fname, 211, mean_labels=5.0)
    fmt = xmc.parse_format(fname)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, num_chunks=k)
    oh = O.OracleHead(W.copy(), fmt_o, k)
    cfg = xmc.SgdSrConfig(lr=lr, weight_decay=1e-4, fmt=fmt, rounding="nearest")
    cfg_o = O.SgdSrConfig(lr=lr, weight_decay=1e-4, fmt=fmt_o, rounding="nearest")
    for step in range(steps):
        xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(0), step)
        O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(0), step)
    got = head.weights.values.float().cpu().numpy()
    assert np.mean(got.view(np.uint32) == oh.values.view(np.uint32)) >= 0.95
    truths = [li[si == i] for i in range(B)]
    ref_scores = oh.scores(X)
    gpu_scores = head.scores(torch.from_numpy(X)).cpu().numpy()
    for kk in (1, 3, 5):
        assert O.dataset_precision_at_k(gpu_scores, truths, kk) == O.dataset_precision_at_k(ref_scores, truths, kk)
    _, labs = head.topk(torch.from_numpy(X), 5)
    labs = labs.cpu().numpy()
    differ = 0
    for s in range(B):
        # the fused top-k ranks the GPU's own scores exactly
        assert np.array_equal(labs[s], O.top_k_indices(gpu_scores[s], 5)), s
        ref = O.top_k_indices(ref_scores[s], 5)
        mine, theirs = set(labs[s].tolist()) - set(ref.tolist()), set(ref.tolist()) - set(labs[s].tolist())
        if not mine:
            continue
        differ += 1
        dz = np.abs(gpu_scores[s] - ref_scores[s])
        for a in mine:
            for b in theirs:
                assert ref_scores[s][b] - ref_scores[s][a] <= dz[a] + dz[b] + 1e-6, (s, a, b)
    assert differ <= 0.05 * B, differ


@pytest.mark.parametrize("fname,rmode", [("e4m3", "stochastic"), ("bf16", "stochastic")])
def test_sr_training_trajectory_matches_oracle(xmc, fname, rmode):
    """splitmix64 SR draws are the reference's own (bit-exact decision given
    the same fp32 update): 4 SR steps along the oracle's trajectory."""
    L, d, B = 2048, 768, 128
    fmt_o, W, X, si, li = _rand_problem(L, d, B, fname, 301, mean_labels=5.0)
    fmt = xmc.parse_format(fname)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, num_chunks=2)
    oh = O.OracleHead(W.copy(), fmt_o, 2)
    cfg = xmc.SgdSrConfig(lr=0.2, weight_decay=1e-4, fmt=fmt, rounding=rmode, sr_impl="splitmix64")
    cfg_o = O.SgdSrConfig(lr=0.2, weight_decay=1e-4, fmt=fmt_o, rounding=rmode)
    Xq = O.round_nearest(fmt_o, X)
    for step in range(4):
        Wb = oh.values.copy()
        head.weights.values.copy_(xmc.cast_native(torch.from_numpy(Wb).cuda(), fmt))
        gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(7), step)
        gx_o = O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(7), step)
        _gx_close(gx.cpu().numpy(), gx_o)
        G = O.logit_gradient(Wb @ Xq.T, si, li, (0, L))
        same, over1, ok = reference_weight_report(head.weights.values.float().cpu().numpy(), oh.values, fmt_o, 0.2,
                                                  G, Xq, sr=True)
        assert same >= 0.995 and ok, (step, same, over1)


@pytest.mark.parametrize("fname,B", [("e4m3", 256), ("bf16", 512), ("bf16", 64)])
def test_subops_take_fp32_G(xmc, fname, B):
    """input_gradient_accumulate / fused_weight_update with the caller's fp32
    G (head.py:199-251): consumed at full precision, like the reference."""
    L, d = 700, 256
    fmt_o, W, X, si, li = _rand_problem(L, d, B, fname, 11)
    oh = O.OracleHead(W.copy(), fmt_o, 1)
    Xq = O.round_nearest(fmt_o, X)
    G = O.logit_gradient(O.head_forward_logits(oh, (0, L), Xq, None, 0), si, li, (0, L))
    acc_ref = O.input_gradient_accumulate(np.zeros((B, d), np.float32), G, oh, (0, L), None, 0)
    fmt = xmc.parse_format(fname)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt)
    acc = torch.zeros((B, d), device="cuda")
    xmc.input_gradient_accumulate(acc, torch.from_numpy(G).cuda(), head, (0, L), None, 0)
    _gx_close(acc.cpu().numpy(), acc_ref)
    cfg_o = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt_o, rounding="nearest")
    O.fused_weight_update(oh, G, Xq, cfg_o, O.RoundingRng(7), 3, (0, L))
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="nearest")
    xmc.fused_weight_update(head, torch.from_numpy(G).cuda(), torch.from_numpy(X), cfg, xmc.RoundingRng(7), 3, (0, L))
    same, over1, ok = reference_weight_report(head.weights.values.float().cpu().numpy(), oh.values, fmt_o, 0.05, G, Xq)
    assert same >= 0.999 and ok, (same, over1)


@pytest.mark.parametrize("fname,kahan,rmode", [("e4m3", "bf16", "stochastic"), ("bf16", "fp32", "nearest")])
def test_head_kahan_reference_precision(xmc, fname, kahan, rmode):
    """Head-Kahan (row A8k) at reference precision against the composed
    oracle with fp32 G, three steps with resync."""
    L, d, B = 700, 256, 128
    fmt_o, W, X, si, li = _rand_problem(L, d, B, fname, 61)
    fmt = xmc.parse_format(fname)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, num_chunks=2, kahan=kahan)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding=rmode, sr_impl="splitmix64")
    oh = O.OracleHead(W.copy(), fmt_o, 2)
    comp = np.zeros((L, d), np.float32)
    cfg_o = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt_o, rounding=rmode)
    cfmt = O.BF16 if kahan == "bf16" else None
    for step in range(3):
        gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(4), step)
        gx_o = O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(4), step, comp=comp, comp_fmt=cfmt)
        _gx_close(gx.cpu().numpy(), gx_o)
        got = head.weights.values.float().cpu().numpy()
        assert np.mean(got.view(np.uint32) == oh.values.view(np.uint32)) >= 0.999
        head.weights.values.copy_(xmc.cast_native(torch.from_numpy(oh.values).cuda(), fmt))
        head.comp.copy_(torch.from_numpy(comp).to(head.comp.dtype).cuda())


def test_head_adamw_reference_precision(xmc):
    L, d, B = 700, 256, 256
    fmt_o, W, X, si, li = _rand_problem(L, d, B, "e4m3", 71)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), xmc.E4M3, num_chunks=2, adamw=True)
    cfg = xmc.KahanAdamWConfig(lr=0.01, beta1=0.9, beta2=0.99, eps=1e-6, weight_decay=0.05, fmt=xmc.E4M3)
    cfg_o = O.KahanAdamWConfig(lr=0.01, beta1=0.9, beta2=0.99, eps=1e-6, weight_decay=0.05, fmt=fmt_o)
    oh = O.OracleHead(W.copy(), fmt_o, 2)
    comp, m, v = (np.zeros((L, d), np.float32) for _ in range(3))
    for step in range(2):
        gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(4), step)
        gx_o = O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(4), step, comp=comp,
                             adam={"m": m, "v": v, "t": step + 1})
        _gx_close(gx.cpu().numpy(), gx_o)
        got = head.weights.values.float().cpu().numpy()
        assert np.mean(got.view(np.uint32) == oh.values.view(np.uint32)) >= 0.999
        np.testing.assert_allclose(head.adam_m.cpu().numpy(), m, rtol=1e-4, atol=1e-6 * np.abs(m).max())
        head.weights.values.copy_(xmc.cast_native(torch.from_numpy(oh.values).cuda(), xmc.E4M3))
        for t_, a_ in ((head.comp, comp), (head.adam_m, m), (head.adam_v, v)):
            t_.copy_(torch.from_numpy(a_).cuda())


def test_c1_exact_shape_kahan(xmc):
    """BASELINE configs[0] at its exact shape: 4,096 labels, d = 768, batch 64,
    bf16, SR + Kahan (bf16 compensation as in PAPER.md:795), 1 chunk -- three
    steps against the composed oracle with fp32 G and the reference's own
    splitmix64 draws."""
    L, d, B = 4096, 768, 64
    fmt_o, W, X, si, li = _rand_problem(L, d, B, "bf16", 401, mean_labels=5.0)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), xmc.BF16, num_chunks=1, kahan="bf16")
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.BF16, rounding="stochastic", sr_impl="splitmix64")
    cfg_o = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt_o, rounding="stochastic")
    oh = O.OracleHead(W.copy(), fmt_o, 1)
    comp = np.zeros((L, d), np.float32)
    for step in range(3):
        Wb = oh.values.copy()
        gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(0), step)
        gx_o = O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(0), step, comp=comp, comp_fmt=O.BF16)
        _gx_close(gx.cpu().numpy(), gx_o)
        got = head.weights.values.float().cpu().numpy()
        assert np.mean(got.view(np.uint32) == oh.values.view(np.uint32)) >= 0.999, step
        # the compensation holds the update's rounding residual: its fp32
        # evaluation-order noise is not rounded away, so bound it instead
        Xq = O.round_nearest(fmt_o, X)
        cg = head.comp.float().cpu().numpy()
        noise = fp32_update_noise(0.05, O.logit_gradient(Wb @ Xq.T, si, li, (0, L)), Xq)
        dw = np.abs(got - oh.values)   # a weight rounded the other way moves its residual by that much
        assert np.all(np.abs(cg - comp) <= dw + O._ulp_of(O.BF16, np.maximum(np.abs(cg), np.abs(comp))) + noise), step
        head.weights.values.copy_(xmc.cast_native(torch.from_numpy(oh.values).cuda(), xmc.BF16))
        head.comp.copy_(torch.from_numpy(comp).to(head.comp.dtype).cuda())


def test_fullsize_c4_grad_x_and_rows_vs_unmodified_reference(xmc):
    """C4 (2,812,281 x 768, batch 256, e4m3, k = 2) at reference precision:
    grad_X against an fp32 restatement over all labels (slabbed G^T W, TF32
    off) at rtol 1e-4, and a row subset of W against the unmodified oracle."""
    L, D, B = 2_812_281, 768, 256
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    W0 = torch.empty((L, D), dtype=torch.float8_e4m3fn, device="cuda")
    for r0 in range(0, L, 262_144):
        r1 = min(L, r0 + 262_144)
        W0[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, D), generator=g, device="cuda") * 0.02, xmc.E4M3)
    rs = np.random.default_rng(3)
    X = rs.normal(size=(B, D)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, 36.17, seed=4)
    Xq = O.round_nearest(O.E4M3, X)
    gx_ref = torch_fp32_grad_x(W0, Xq, si, li).cpu().numpy()
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W0.clone(), xmc.E4M3), num_chunks=2)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding="stochastic", sr_impl="splitmix64")
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(11), 0).cpu().numpy()
    _gx_close(gx, gx_ref)
    rows = set(rs.choice(L, 400, replace=False).tolist()) | set(np.unique(li)[:100].tolist())
    rows |= {0, 127, 128, L // 2 - 1, L // 2, L - 1}
    rows = np.array(sorted(rows), dtype=np.int64)
    w0 = W0[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    z = w0 @ Xq.T
    pos = np.zeros_like(z, dtype=bool)
    idx = {r: i for i, r in enumerate(rows)}
    for s, l in zip(si, li):
        if int(l) in idx:
            pos[idx[int(l)], s] = True
    G = O.logit_gradient(z, np.nonzero(pos)[1], np.nonzero(pos)[0], (0, len(rows)))
    cfg_o = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=O.E4M3, rounding="stochastic")
    gidx = rows[:, None].astype(np.uint64) * np.uint64(D) + np.arange(D, dtype=np.uint64)[None, :]
    ref = O.sgd_sr_values(w0, G @ Xq, cfg_o, O.RoundingRng(11), 0, O.HEAD_WEIGHTS_TAG, gidx)
    got = head.weights.values[torch.from_numpy(rows).cuda()].float().cpu().numpy()
    same, over1, ok = reference_weight_report(got, ref, O.E4M3, 0.05, G, Xq, sr=True)
    assert same >= 0.999 and ok, (same, over1)


@pytest.mark.parametrize("fname,d,B,extra", [("e4m3", 32, 32, None), ("bf16", 32, 64, "kahan"), ("e4m3", 96, 256, "dropout"),
                                             ("bf16", 160, 128, None), ("e4m3", 800, 128, "kahan")])
def test_partial_d_tiles(xmc, fname, d, B, extra):
    """d a multiple of 32 but not of 128 (the reference takes any d; the
    kernels need d % 32 == 0): the last 128-column tile is zero-filled by TMA
    on load and clipped on store, the per-thread side buffers (compensation,
    keep bits, grad_X rows) skip the columns past d."""
    L = 900
    fmt_o, W, X, si, li = _rand_problem(L, d, B, fname, 501)
    fmt = xmc.parse_format(fname)
    p = 0.2 if extra == "dropout" else 0.0
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, num_chunks=2, dropout_p=p,
                                      kahan="bf16" if extra == "kahan" else None)
    oh = O.OracleHead(W.copy(), fmt_o, 2, dropout_p=p)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic", sr_impl="splitmix64")
    cfg_o = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt_o, rounding="stochastic")
    comp = np.zeros((L, d), np.float32) if extra == "kahan" else None
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(3), 1)
    gx_o = O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(3), 1, comp=comp,
                         comp_fmt=O.BF16 if extra == "kahan" else None)
    _gx_close(gx.cpu().numpy(), gx_o)
    got = head.weights.values.float().cpu().numpy()
    assert np.mean(got.view(np.uint32) == oh.values.view(np.uint32)) >= 0.999
    if extra == "kahan":
        assert np.isfinite(head.comp.float().cpu().numpy()).all()
    # the operand mode on the same shape (oracle given the same operand G)
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, num_chunks=2, dropout_p=p, precision="operand")
    oh = O.OracleHead(W.copy(), fmt_o, 2, dropout_p=p)
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(3), 1)
    gx_o = O.head_update(oh, X, si, li, cfg_o, O.RoundingRng(3), 1, g_quant=True)
    _gx_close(gx.cpu().numpy(), gx_o)
    assert np.mean(head.weights.values.float().cpu().numpy().view(np.uint32) == oh.values.view(np.uint32)) >= 0.99
    # scores / fused top-k on the partial tile
    sc = head.scores(torch.from_numpy(X)).cpu().numpy()
    np.testing.assert_allclose(sc, oh.scores(X), rtol=1e-5, atol=1e-5)
    _, labs = head.topk(torch.from_numpy(X), 3)
    for s in range(B):
        assert np.array_equal(labs[s].cpu().numpy(), O.top_k_indices(sc[s], 3))
