"""CPU restatement of the reference's training loop around the head --
TEST INFRASTRUCTURE ONLY (same rules as lpxmc_oracle.py: only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may use it).

Restates, from /root/reference/pkg/src/lpxmc:
  * data.py:26-45 SparseDataset, :144-199 SyntheticSpec / generate_synthetic;
  * trainer.py:41-70 TrainConfig, :73-111 TinyEncoder, :171-286 Trainer
    (held-out split, warmup, the head step with the mean-|G| divergence proxy
    and the frozen lr = 0 path, encoder Kahan-AdamW, run_epoch, evaluate).

The head half of Trainer.step is injectable (``head_step``), so the same loop
drives either the oracle head (lpxmc_oracle.head_update, the reference
itself) or the GPU head (paper_2510_11168_b200.trainer_hooks) -- the F2
"trainer integration" parity of SURVEY.md 8(f).  Pinned bit-exactly against
golden runs of the reference Trainer (tests/golden/make_trainer_golden.py,
tests/test_oracle_trainer.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import lpxmc_oracle as O

_SPLIT_TAG = O.tensor_tag("trainer.split")   # trainer.py:32
_DIVERGENCE_LEVEL = 0.999                     # trainer.py:36-37
_DIVERGENCE_PATIENCE = 100


class DivergenceError(RuntimeError):          # trainer.py:40-43
    def __init__(self, step: int, message: str):
        super().__init__(f"training diverged at step {step}: {message}")
        self.step = step


@dataclass
class SparseDataset:                           # data.py:26-45
    num_samples: int
    num_features: int
    num_labels: int
    labels: list
    features: list
    values: list

    def dense_features(self, idx):
        out = np.zeros((len(idx), self.num_features), dtype=np.float32)
        for row, i in enumerate(idx):
            out[row, self.features[i]] = self.values[i]
        return out


@dataclass
class SyntheticSpec:                           # data.py:144-154
    num_samples: int
    num_features: int
    num_labels: int
    mean_labels: float = 2.0
    zipf_exponent: float = 1.0
    noise: float = 0.1
    min_labels: int = 0
    seed: int = 0


def generate_synthetic(spec: SyntheticSpec) -> SparseDataset:
    """data.py:169-199."""
    rng = np.random.default_rng(spec.seed)
    freqs = np.arange(1, spec.num_labels + 1, dtype=np.float64) ** -spec.zipf_exponent
    freqs /= freqs.sum()
    protos = rng.normal(size=(spec.num_labels, spec.num_features)).astype(np.float32)
    protos /= np.linalg.norm(protos, axis=1, keepdims=True)
    labels, features, values = [], [], []
    for _ in range(spec.num_samples):
        count = min(max(spec.min_labels, rng.poisson(spec.mean_labels)), spec.num_labels)
        ls = rng.choice(spec.num_labels, size=count, replace=False, p=freqs)
        ls = np.sort(ls.astype(np.int64))
        if count:
            x = protos[ls].mean(axis=0) + rng.normal(scale=spec.noise, size=spec.num_features).astype(np.float32)
        else:
            x = rng.normal(scale=spec.noise, size=spec.num_features).astype(np.float32)
        labels.append(ls)
        features.append(np.arange(spec.num_features, dtype=np.int64))
        values.append(x.astype(np.float32))
    return SparseDataset(spec.num_samples, spec.num_features, spec.num_labels, labels, features, values)


@dataclass
class TrainConfig:                             # trainer.py:46-70
    hidden: int = 64
    embed_dim: int = 32
    head_format: str = "fp32"
    encoder_format: str = "fp32"
    head_lr: float = 0.1
    encoder_lr: float = 1e-3
    head_weight_decay: float = 0.0
    encoder_weight_decay: float = 0.01
    head_rounding: str = "stochastic"
    warmup_steps: int = 0
    epochs: int = 10
    batch_size: int = 32
    chunks: int = 1
    dropout_p: float = 0.0
    grad_clip: float | None = None
    eval_fraction: float = 0.2
    seed: int = 0

    def head_fmt(self):
        return O.parse_format(self.head_format)

    def encoder_fmt(self):
        return O.parse_format(self.encoder_format)


class _Param:
    """KahanAdamWParam (optimizers.py:94-109): sum, comp, m, v."""

    def __init__(self, values, fmt):
        self.values = O.round_nearest(fmt, values)
        self.comp = np.zeros_like(self.values)
        self.m = np.zeros_like(self.values)
        self.v = np.zeros_like(self.values)


class TinyEncoder:                             # trainer.py:73-111
    def __init__(self, num_features, hidden, embed_dim, fmt, seed):
        g = np.random.default_rng(seed)

        def init(shape, scale):
            return g.normal(scale=scale, size=shape).astype(np.float32)
        self.params = {
            "w1": _Param(init((num_features, hidden), 1.0 / np.sqrt(num_features)), fmt),
            "b1": _Param(np.zeros(hidden, np.float32), fmt),
            "w2": _Param(init((hidden, embed_dim), 1.0 / np.sqrt(hidden)), fmt),
            "b2": _Param(np.zeros(embed_dim, np.float32), fmt),
        }

    def forward(self, x):
        z = x @ self.params["w1"].values + self.params["b1"].values
        h = np.maximum(z, np.float32(0))
        emb = h @ self.params["w2"].values + self.params["b2"].values
        return emb, (x, z, h)

    def backward(self, cache, d_emb):
        x, z, h = cache
        dw2 = h.T @ d_emb
        db2 = d_emb.sum(axis=0)
        dh = d_emb @ self.params["w2"].values.T
        dz = dh * (z > 0)
        dw1 = x.T @ dz
        db1 = dz.sum(axis=0)
        return {"w1": dw1, "b1": db1, "w2": dw2, "b2": db2}


def oracle_head_step(trainer, emb, rows, cols, head_lr):
    """The head half of Trainer.step on the oracle head (trainer.py:176-205):
    returns (d_emb, sum |G|, number of G entries)."""
    cfg = trainer.cfg
    gsum = [0.0, 0]

    def stat_probe(step, chunk, G):
        gsum[0] += float(np.abs(G, dtype=np.float64).sum())
        gsum[1] += G.size

    if head_lr > 0:
        hcfg = O.SgdSrConfig(lr=head_lr, weight_decay=cfg.head_weight_decay, fmt=cfg.head_fmt(),
                             rounding=cfg.head_rounding)
        d_emb = O.head_update(trainer.head, emb, rows, cols, hcfg, trainer.rng, trainer.global_step,
                              probe=stat_probe)
    else:
        frozen = O.SgdSrConfig(lr=1.0, fmt=cfg.head_fmt(), rounding="nearest")
        before = trainer.head.values.copy()
        d_emb = O.head_update(trainer.head, emb, rows, cols, frozen, trainer.rng, trainer.global_step,
                              probe=stat_probe)
        trainer.head.values[...] = before
        d_emb[...] = 0.0
    return d_emb, gsum[0], gsum[1]


class Trainer:                                 # trainer.py:171-251
    def __init__(self, dataset, cfg: TrainConfig, head_step=oracle_head_step):
        self.dataset = dataset
        self.cfg = cfg
        self.rng = O.RoundingRng(cfg.seed)
        self.head = O.OracleHead.create(dataset.num_labels, cfg.embed_dim, cfg.head_fmt(), seed=cfg.seed,
                                        num_chunks=cfg.chunks, dropout_p=cfg.dropout_p)
        self.encoder = TinyEncoder(dataset.num_features, cfg.hidden, cfg.embed_dim, cfg.encoder_fmt(),
                                   cfg.seed + 1)
        self.adamw = O.KahanAdamWConfig(lr=cfg.encoder_lr, weight_decay=cfg.encoder_weight_decay,
                                        fmt=cfg.encoder_fmt())
        self.head_step = head_step
        self.global_step = 0
        self.epoch = 0
        self.history = []
        self.mean_g = []
        self._hot_steps = 0
        u = self.rng.uniform(0, _SPLIT_TAG, np.arange(dataset.num_samples, dtype=np.uint64))
        held = u < cfg.eval_fraction
        self.eval_idx = np.flatnonzero(held)
        self.train_idx = np.flatnonzero(~held)

    def _lr_scale(self):                       # trainer.py:157-161
        if self.cfg.warmup_steps <= 0:
            return 1.0
        return min(1.0, self.global_step / self.cfg.warmup_steps)

    def step(self, batch_idx):                 # trainer.py:168-226
        self.global_step += 1
        xf = self.dataset.dense_features(batch_idx)
        emb, cache = self.encoder.forward(xf)
        rows, cols = [], []
        for r, i in enumerate(batch_idx):
            ls = self.dataset.labels[i]
            rows.extend([r] * len(ls))
            cols.extend(ls.tolist())
        rows, cols = np.array(rows, np.int64), np.array(cols, np.int64)
        scale = self._lr_scale()
        head_lr = self.cfg.head_lr * scale if self.cfg.head_lr > 0 else 0.0
        d_emb, gs, gn = self.head_step(self, emb, rows, cols, head_lr)
        d_emb = np.asarray(d_emb, dtype=np.float32)
        mean_g = gs / max(gn, 1)
        self.mean_g.append(mean_g)
        if not np.isfinite(mean_g):
            raise DivergenceError(self.global_step, "non-finite logit gradients")
        self._hot_steps = self._hot_steps + 1 if mean_g > _DIVERGENCE_LEVEL else 0
        if self._hot_steps >= _DIVERGENCE_PATIENCE:
            raise DivergenceError(self.global_step, "logit gradients saturated (mean |g| > 0.999)")
        grads = self.encoder.backward(cache, d_emb)
        if self.cfg.grad_clip is not None:
            norm = np.sqrt(sum(float((g.astype(np.float64) ** 2).sum()) for g in grads.values()))
            if norm > self.cfg.grad_clip:
                factor = np.float32(self.cfg.grad_clip / norm)
                grads = {k: g * factor for k, g in grads.items()}
        enc_lr = self.cfg.encoder_lr * scale
        for name, g in grads.items():
            p = self.encoder.params[name]
            p.values, p.comp, p.m, p.v = O.kahan_adamw_values(p.values, p.comp, p.m, p.v, g, self.adamw,
                                                              self.global_step, lr=enc_lr)
        return mean_g

    def run_epoch(self):                       # trainer.py:228-238
        order = np.random.default_rng((self.cfg.seed, self.epoch)).permutation(self.train_idx)
        bs = self.cfg.batch_size
        for i in range(0, len(order), bs):
            self.step(order[i:i + bs])
        self.epoch += 1
        record = {"epoch": self.epoch, "step": self.global_step}
        record.update(self.evaluate())
        self.history.append(record)
        return record

    def predict_scores(self, idx, scores_fn=None):   # trainer.py:240-243
        xf = self.dataset.dense_features(idx)
        emb, _ = self.encoder.forward(xf)
        return self.head.scores(emb) if scores_fn is None else scores_fn(emb)

    def evaluate(self, ks=(1, 3, 5)):          # trainer.py:245-251
        idx = self.eval_idx if self.eval_idx.size else self.train_idx
        scores = self.predict_scores(idx, getattr(self, "scores_fn", None))
        truths = [self.dataset.labels[i] for i in idx]
        return {f"p_at_{k}": O.dataset_precision_at_k(scores, truths, k) for k in ks if k <= self.dataset.num_labels}
