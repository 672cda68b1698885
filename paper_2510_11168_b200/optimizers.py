"""SGD with one rounding onto the storage grid -- mirror of lpxmc.optimizers.

``SgdSrConfig`` keeps the reference fields and validation
(optimizers.py:28-41) and adds ``sr_impl``: the draw generator used when
``rounding == "stochastic"``.

* ``"hash"`` (default, the fast product path): keyed random words fed to the
  sm_100a hardware stochastic-rounding conversion (cvt.rs); word i of a step
  is a stateless PCG hash (RXS-M-XS) of i + key(seed, step, tensor_id), the
  same keyed-hash construction as the reference's splitmix64 draws
  (rng.py:36-57) at a quarter of Philox's instruction cost.  SR decisions
  match the reference in distribution (unbiased, same variance).
* ``"philox"``: the same conversion with Philox4x32-7 words.
* ``"splitmix64"``: the reference's own keyed generator (rng.py:36-57) and
  fp64 neighbour/probability comparison (formats.py:209-225).  Given the same
  fp32 update value the decision is bit-identical to the reference.

``sgd_sr_step`` (optimizers.py:51-74) runs elementwise on the GPU on
float32 on-grid values, bit-exact with the reference for both rounding modes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib
from .formats import FP32, FloatFormat, _f32_cuda, _index_tensor


@dataclass
class SgdSrConfig:
    lr: float
    weight_decay: float = 0.0
    fmt: FloatFormat = field(default_factory=lambda: FP32)
    rounding: str = "stochastic"  # or "nearest"
    sr_impl: str = "hash"         # or "philox", or "splitmix64" (bit-exact reference draws)

    def __post_init__(self):
        if self.lr <= 0:
            raise ValueError("lr must be positive")
        if self.weight_decay < 0:
            raise ValueError("weight_decay must be non-negative")
        if self.rounding not in ("stochastic", "nearest"):
            raise ValueError(f"unknown rounding mode {self.rounding!r}")
        if self.sr_impl not in ("hash", "philox", "splitmix64"):
            raise ValueError(f"unknown SR generator {self.sr_impl!r}")

    @property
    def rounding_code(self) -> int:
        if self.rounding == "nearest":
            return _lib.ROUND_NEAREST
        return _lib.ROUND_SR_EXACT if self.sr_impl == "splitmix64" else _lib.ROUND_SR_FAST

    @property
    def sr_bits(self) -> int:
        """xmc_step_args.sr_bits: the SR_FAST word generator (0 hash, 1 Philox)."""
        return 1 if self.sr_impl == "philox" else 0


def sgd_sr_step(w: torch.Tensor, grad, cfg: SgdSrConfig, rng, step: int, tensor_id: int = 0,
                global_index=None) -> torch.Tensor:
    """w <- ROUND(w - lr*(grad + wd*w)), in place on a float32 CUDA tensor of
    on-grid values (optimizers.py:51-74).  Stochastic rounding always uses the
    reference's splitmix64 keys here (bit-exact)."""
    if not (w.is_cuda and w.dtype == torch.float32 and w.is_contiguous()):
        raise ValueError("w must be a contiguous float32 CUDA tensor")
    g = _f32_cuda(grad)
    if tuple(g.shape) != tuple(w.shape):
        raise ValueError(f"shape mismatch: weights {tuple(w.shape)}, grad {tuple(g.shape)}")
    idx = _index_tensor(global_index, w.numel(), w.device)
    rmode = _lib.ROUND_NEAREST if cfg.rounding == "nearest" else _lib.ROUND_SR_EXACT
    _lib.check(_lib.load().xmc_sgd_sr_step(
        cfg.fmt.grid(), w.data_ptr(), g.data_ptr(), w.numel(), cfg.lr, cfg.weight_decay, rmode,
        rng.seed, step & (2**64 - 1), tensor_id & (2**64 - 1), _lib.ptr(idx), None,
        _lib.stream_ptr()))
    return w


def kahan_sgd_step(w: torch.Tensor, comp: torch.Tensor, grad, cfg: SgdSrConfig, rng, step: int,
                   tensor_id: int = 0, global_index=None):
    """Head-Kahan SGD: kahan_add (formats.py:246-263) of the
    SGD update onto the grid, ROUND = RTN or keyed SR; float32 w and comp."""
    for t in (w, comp):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError("w and comp must be contiguous float32 CUDA tensors")
    g = _f32_cuda(grad)
    if tuple(g.shape) != tuple(w.shape) or tuple(comp.shape) != tuple(w.shape):
        raise ValueError("shape mismatch")
    idx = _index_tensor(global_index, w.numel(), w.device)
    rmode = _lib.ROUND_NEAREST if cfg.rounding == "nearest" else _lib.ROUND_SR_EXACT
    _lib.check(_lib.load().xmc_kahan_sgd_step(
        cfg.fmt.grid(), w.data_ptr(), comp.data_ptr(), g.data_ptr(), w.numel(), cfg.lr,
        cfg.weight_decay, rmode, rng.seed, step & (2**64 - 1), tensor_id & (2**64 - 1),
        _lib.ptr(idx), None, _lib.stream_ptr()))
    return w, comp


@dataclass
class KahanAdamWConfig:
    """optimizers.py:77-91 (same fields and validation)."""
    lr: float
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    fmt: FloatFormat = field(default_factory=lambda: FP32)

    def __post_init__(self):
        if not (0.0 <= self.beta1 < 1.0 and 0.0 <= self.beta2 < 1.0):
            raise ValueError("betas must lie in [0, 1)")
        if self.eps <= 0:
            raise ValueError("eps must be positive")


class KahanAdamWParam:
    """One parameter tensor with its compensation buffer and moments
    (optimizers.py:93-109), as float32 CUDA tensors: ``sum`` holds on-grid
    values, ``comp`` the Kahan compensation, ``m`` / ``v`` the moments."""

    def __init__(self, sum_: torch.Tensor, comp: torch.Tensor, m: torch.Tensor, v: torch.Tensor):
        for t in (sum_, comp, m, v):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
                raise ValueError("parameter state must be contiguous float32 CUDA tensors")
            if t.shape != sum_.shape:
                raise ValueError("parameter state shapes differ")
        self.sum, self.comp, self.m, self.v = sum_, comp, m, v

    @classmethod
    def from_values(cls, values, fmt: FloatFormat) -> "KahanAdamWParam":
        from .formats import round_nearest
        vals = round_nearest(fmt, _f32_cuda(values).clone())
        return cls(vals, torch.zeros_like(vals), torch.zeros_like(vals), torch.zeros_like(vals))

    @property
    def values(self) -> torch.Tensor:
        return self.sum


def kahan_adamw_step(param: KahanAdamWParam, grad, cfg: KahanAdamWConfig, t: int, lr: float | None = None) -> None:
    """In-place AdamW step with Kahan-compensated parameter accumulation
    (optimizers.py:112-137; kahan_add formats.py:246-263), bit-exact with the
    reference.  ``lr`` overrides cfg.lr (warmup schedules).  Raises ValueError
    on non-finite moments or updates, leaving the state unchanged."""
    if t < 1:
        raise ValueError("step index t must be >= 1")
    g = _f32_cuda(grad)
    if tuple(g.shape) != tuple(param.values.shape):
        raise ValueError("gradient shape mismatch")
    _lib.check(_lib.load().xmc_kahan_adamw_step(
        cfg.fmt.grid(), param.sum.data_ptr(), param.comp.data_ptr(), param.m.data_ptr(), param.v.data_ptr(),
        g.data_ptr(), param.sum.numel(), float(cfg.lr if lr is None else lr), float(cfg.beta1),
        float(cfg.beta2), float(cfg.eps), float(cfg.weight_decay), int(t), _lib.stream_ptr()))
