"""Trainer integration: the reference's training loop
(oracle/lpxmc_trainer_oracle.py, pinned bit-exactly to lpxmc's Trainer by
tests/test_oracle_trainer.py) driving the GPU head through
paper_2510_11168_b200.trainer_hooks.HeadTrainerStep -- the head half of
Trainer.step (trainer.py:168-226): warmup, the mean-|G| divergence proxy from
the fused forward's statistics, the frozen lr = 0 path -- and reference
acceptance 09 (test_acceptance.py:227-241: e4m3 + SR head reaches P@1 >= 0.90
on the frozen EASY benchmark within 25 epochs) with the GPU head, in both
backward precisions."""

import numpy as np
import pytest
import torch

from oracle import lpxmc_oracle as O
from oracle import lpxmc_trainer_oracle as T

pytestmark = pytest.mark.gpu

EASY_SPEC = dict(num_samples=640, num_features=32, num_labels=32, mean_labels=1.0, min_labels=1, noise=0.05, seed=7)
EASY_CFG = dict(hidden=64, embed_dim=32, head_lr=0.3, encoder_lr=3e-3, epochs=25, batch_size=32, chunks=1, seed=1)


@pytest.fixture(scope="module")
def xmc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11168_b200 as xmc
    return xmc


def _gpu_trainer(xmc, cfg, precision, sr_impl="hash"):
    from paper_2510_11168_b200.trainer_hooks import HeadTrainerStep
    ds = T.generate_synthetic(T.SyntheticSpec(**EASY_SPEC))
    fmt = xmc.parse_format(cfg.head_format)
    head = xmc.ChunkedHead.create(ds.num_labels, cfg.embed_dim, fmt, seed=cfg.seed, num_chunks=cfg.chunks,
                                  precision=precision)
    hs = HeadTrainerStep(head, fmt, cfg.head_lr, cfg.head_weight_decay, cfg.head_rounding, cfg.warmup_steps,
                         sr_impl=sr_impl)
    rng = xmc.RoundingRng(cfg.seed)

    def head_step(trainer, emb, rows, cols, head_lr):
        d_emb, mean_g = hs(emb, rows, cols, rng, trainer.global_step)
        n = head.num_labels * emb.shape[0]
        return d_emb.cpu().numpy(), mean_g * n, n

    t = T.Trainer(ds, cfg, head_step=head_step)
    t.scores_fn = lambda emb: hs.scores(emb).cpu().numpy()
    return t, head, hs


@pytest.mark.parametrize("fmt,rounding,precision", [("e4m3", "stochastic", "reference"), ("bf16", "nearest", "reference"),
                                                    ("e4m3", "stochastic", "operand")])
def test_first_steps_match_oracle_trainer(xmc, fmt, rounding, precision):
    """From the same initial state the GPU head's step gives the reference
    step's mean |G| (fp32 tolerance) and input gradient; three steps with
    the oracle head state copied back into the GPU head between steps."""
    cfg = T.TrainConfig(**{**EASY_CFG, "head_format": fmt, "head_rounding": rounding, "warmup_steps": 3,
                           "chunks": 2})
    ds = T.generate_synthetic(T.SyntheticSpec(**EASY_SPEC))
    ref = T.Trainer(ds, cfg)
    gpu, head, hs = _gpu_trainer(xmc, cfg, precision, sr_impl="splitmix64")
    assert np.array_equal(head.weights.values.float().cpu().numpy(), ref.head.values)
    order = np.random.default_rng((cfg.seed, 0)).permutation(ref.train_idx)
    for s in range(3):
        idx = order[s * 32:(s + 1) * 32]
        ref.step(idx)
        gpu.step(idx)
        np.testing.assert_allclose(gpu.mean_g[-1], ref.mean_g[-1], rtol=1e-5)
        # resync the head so the next step starts from the same state
        head.weights.values.copy_(xmc.cast_native(torch.from_numpy(ref.head.values).cuda(), head.fmt))
        for name in ref.encoder.params:
            gp, rp = gpu.encoder.params[name], ref.encoder.params[name]
            gp.values, gp.comp, gp.m, gp.v = rp.values.copy(), rp.comp.copy(), rp.m.copy(), rp.v.copy()


def test_frozen_lr0_path_leaves_weights_bit_identical(xmc):
    """trainer.py:196-205: head_lr = 0 runs an lr = 1 RTN pass for the
    statistics, restores W bit for bit and zeroes the input gradient."""
    cfg = T.TrainConfig(**{**EASY_CFG, "head_format": "e4m3", "head_lr": 0.0})
    gpu, head, hs = _gpu_trainer(xmc, cfg, "reference")
    ds = T.generate_synthetic(T.SyntheticSpec(**EASY_SPEC))
    ref = T.Trainer(ds, cfg)
    w0 = head.weights.values.clone()
    idx = ref.train_idx[:32]
    emb, _ = gpu.encoder.forward(ds.dense_features(idx))
    rows = np.concatenate([[r] * len(ds.labels[i]) for r, i in enumerate(idx)]).astype(np.int64)
    cols = np.concatenate([ds.labels[i] for i in idx]).astype(np.int64)
    d_emb, mean_g = hs(emb, rows, cols, xmc.RoundingRng(cfg.seed), 1)
    assert torch.equal(head.weights.values.view(torch.uint8), w0.view(torch.uint8))
    assert torch.count_nonzero(d_emb) == 0
    ref.global_step = 1
    _, gs, gn = T.oracle_head_step(ref, emb, rows, cols, 0.0)
    np.testing.assert_allclose(mean_g, gs / gn, rtol=1e-5)
    for s in range(3):   # the whole loop: the encoder trains, the head never moves
        gpu.step(ref.train_idx[32 * (s + 1):32 * (s + 2)])
    assert torch.equal(head.weights.values.view(torch.uint8), w0.view(torch.uint8))


def test_divergence_proxy_raises(xmc):
    """Saturated logits (every |G| ~ 1) for 100 consecutive steps raise
    DivergenceError like trainer.py:208-213."""
    from paper_2510_11168_b200.trainer_hooks import DivergenceError, HeadTrainerStep
    L, d, B = 64, 32, 32
    head = xmc.ChunkedHead.from_float(torch.full((L, d), 8.0), xmc.E4M3)
    hs = HeadTrainerStep(head, xmc.E4M3, 1e-6, rounding="nearest")
    X = np.ones((B, d), np.float32)
    with pytest.raises(DivergenceError):
        for s in range(1, 120):
            _, mean_g = hs(X, np.zeros(0, np.int64), np.zeros(0, np.int64), xmc.RoundingRng(0), s)
            assert mean_g > 0.999
    assert hs.hot_steps == 100


@pytest.mark.parametrize("precision", ["reference", "operand"])
def test_acceptance_09_learnability_with_gpu_head(xmc, precision):
    """Reference acceptance 09 (test_acceptance.py:227-241) with the GPU
    head: e4m3 + SR (production hash words), 25 epochs on the frozen EASY
    benchmark, final P@1 >= 0.90.  The oracle's own e4m3 + SR run of the same
    config is reported beside it."""
    cfg = T.TrainConfig(**{**EASY_CFG, "head_format": "e4m3", "head_rounding": "stochastic"})
    gpu, head, hs = _gpu_trainer(xmc, cfg, precision)
    for _ in range(cfg.epochs):
        rec = gpu.run_epoch()
    assert rec["p_at_1"] >= 0.90, rec
    print(f"acceptance 09, GPU e4m3+SR head ({precision} precision): {rec}")
