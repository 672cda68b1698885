"""The head half of the reference's training step on the GPU head
(lpxmc.trainer.Trainer.step, trainer.py:168-226) -- the drop-in for a caller
that keeps its own encoder (numpy, torch, ...) and hands the head its batch
embeddings.

Per step (global_step is 1-based, as Trainer.step increments it first):
  * warmup: lr scale min(1, global_step / warmup_steps) (trainer.py:157-161),
    head lr = head_lr * scale if head_lr > 0 else 0 (:188-189);
  * head_lr > 0: head_update with the fused step; sum |G| comes from the
    forward epilogue (ChunkedHead.collect_stats), so the divergence proxy
    mean |G| = sum |G| / (L * B) costs no extra pass (:182-186, :207);
  * head_lr == 0: the frozen pass -- an lr = 1 RTN step whose weights are
    restored bit for bit, input gradient zeroed (:196-205);
  * divergence: non-finite mean |G| raises DivergenceError at once; mean |G|
    above 0.999 for 100 consecutive steps raises it too (:208-213).
"""

from __future__ import annotations

import math

import torch

from .formats import FloatFormat
from .head import BatchInput, ChunkedHead, head_update
from .optimizers import SgdSrConfig

DIVERGENCE_LEVEL = 0.999      # trainer.py:36-37
DIVERGENCE_PATIENCE = 100


class DivergenceError(RuntimeError):
    """trainer.py:40-43."""

    def __init__(self, step: int, message: str):
        super().__init__(f"training diverged at step {step}: {message}")
        self.step = step


class HeadTrainerStep:
    """Callable doing the head part of one training step.

    ``step(emb, sample_idx, label_idx, rng, global_step)`` returns
    ``(d_emb, mean_g)``: the input gradient (B, d) fp32 on the head's device
    and the mean |logit gradient| of the step (a Python float; reading it
    synchronises the stream, as the reference's proxy needs the value)."""

    def __init__(self, head: ChunkedHead, fmt: FloatFormat, head_lr: float, weight_decay: float = 0.0,
                 rounding: str = "stochastic", warmup_steps: int = 0, sr_impl: str = "hash"):
        self.head = head
        self.fmt = fmt
        self.head_lr = float(head_lr)
        self.weight_decay = float(weight_decay)
        self.rounding = rounding
        self.warmup_steps = int(warmup_steps)
        self.sr_impl = sr_impl
        self.hot_steps = 0
        head.collect_stats = True

    def lr_scale(self, global_step: int) -> float:
        if self.warmup_steps <= 0:
            return 1.0
        return min(1.0, global_step / self.warmup_steps)

    def __call__(self, emb, sample_idx, label_idx, rng, global_step: int):
        head = self.head
        batch = BatchInput(emb, sample_idx, label_idx)
        scale = self.lr_scale(global_step)
        lr = self.head_lr * scale if self.head_lr > 0 else 0.0
        if lr > 0:
            cfg = SgdSrConfig(lr=lr, weight_decay=self.weight_decay, fmt=self.fmt, rounding=self.rounding,
                              sr_impl=self.sr_impl)
            d_emb = head_update(head, batch, cfg, rng, global_step)
        else:
            frozen = SgdSrConfig(lr=1.0, fmt=self.fmt, rounding="nearest")
            before = head.weights.values.clone()
            comp = head.comp.clone() if head.comp is not None else None
            d_emb = head_update(head, batch, frozen, rng, global_step)
            head.weights.values.copy_(before)
            if comp is not None:
                head.comp.copy_(comp)
            d_emb.zero_()
        b = d_emb.shape[0]
        mean_g = float(head.last_stats[0].item()) / max(head.num_labels * b, 1)
        if not math.isfinite(mean_g):
            raise DivergenceError(global_step, "non-finite logit gradients")
        self.hot_steps = self.hot_steps + 1 if mean_g > DIVERGENCE_LEVEL else 0
        if self.hot_steps >= DIVERGENCE_PATIENCE:
            raise DivergenceError(global_step, "logit gradients saturated (mean |g| > 0.999)")
        return d_emb, mean_g

    def scores(self, emb) -> torch.Tensor:
        """Trainer.predict_scores' head part (trainer.py:240-243)."""
        return self.head.scores(emb)
