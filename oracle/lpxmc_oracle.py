"""CPU oracle for the ELMO chunked-head hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``lpxmc``
(``/root/reference/pkg/src/lpxmc``) restricted to the hot path named by
BASELINE.json's north_star: the chunked head step ``head_update`` and every
function it calls (rounding grids, keyed RNG, SGD+rounding, Kahan add), plus
the scoring/top-k judge used for P@k parity.  Every function cites the
reference file:line it follows.

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs -- as the CHECKER or the timed
CPU baseline only.  The product package ``paper_2510_11168_b200`` never
imports it; its GPU path fails loudly when the CUDA library is missing.

Parity pinning: the rounding, RNG, SGD-update, Kahan and partition functions
are checked BIT-EXACT against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports lpxmc from /root/reference in the
build container; the vectors are committed as ``tests/golden/*.npz``).  GEMM-
derived values (logits, G, grad_X, updated weights) are pinned within fp32
tolerance because the reference's fp32 accumulation order is OpenBLAS-defined
(SURVEY.md section 8(c)).

Differences from the reference that do not change results:
  * the SR / RTN rounding is vectorised over a whole canonical piece instead
    of the reference's 64x64 Python block loop (rounding is elementwise and
    keyed by the global flat index, so the block order is irrelevant,
    head.py:230-248);
  * the per-block scratch GEMM ``g_rows @ Xq[:, c0:c1]`` is kept per 64-row
    block x full-width columns; each element is still one fp32 dot product
    over the batch dimension.
"""

from __future__ import annotations

from dataclasses import dataclass, field
import re
import struct

import numpy as np

# ---------------------------------------------------------------------------
# formats.py restatement


@dataclass(frozen=True)
class FloatFormat:
    """Emulated float grid (E, M).  formats.py:49-137."""

    exp_bits: int
    man_bits: int
    saturating: bool = True
    extended_range: bool | None = field(default=None)

    def __post_init__(self):  # formats.py:59-67
        if not (2 <= self.exp_bits <= 8):
            raise ValueError(f"exp_bits must be in [2, 8], got {self.exp_bits}")
        if not (0 <= self.man_bits <= 23):
            raise ValueError(f"man_bits must be in [0, 23], got {self.man_bits}")
        if self.extended_range is None:
            object.__setattr__(self, "extended_range",
                               (self.exp_bits, self.man_bits) == (4, 3))

    @property
    def bias(self) -> int:  # formats.py:69-71
        return 2 ** (self.exp_bits - 1) - 1

    @property
    def min_normal_exp(self) -> int:  # formats.py:73-75
        return 1 - self.bias

    @property
    def max_exp(self) -> int:  # formats.py:77-79
        return self.bias + 1 if self.extended_range else self.bias

    @property
    def min_exp(self) -> int:  # formats.py:81-84
        return self.min_normal_exp - self.man_bits

    @property
    def max_finite(self) -> float:  # formats.py:86-94
        if self.extended_range:
            if self.man_bits == 0:
                raise ValueError("extended range needs at least one mantissa bit")
            top = 2.0 - 2.0 ** (1 - self.man_bits)
        else:
            top = 2.0 - 2.0 ** (-self.man_bits)
        return float(np.ldexp(top, self.max_exp))

    @property
    def storage_bits(self) -> int:  # formats.py:100-102
        return 1 + self.exp_bits + self.man_bits

    @property
    def name(self) -> str:  # formats.py:108-113
        named = {(8, 23): "fp32", (8, 7): "bf16", (5, 10): "fp16",
                 (4, 3): "e4m3", (5, 2): "e5m2"}
        return named.get((self.exp_bits, self.man_bits),
                         f"e{self.exp_bits}m{self.man_bits}")

    @property
    def is_working_precision(self) -> bool:  # formats.py:115-118
        return self.exp_bits == 8 and self.man_bits == 23


FP32 = FloatFormat(8, 23)   # formats.py:139-143
BF16 = FloatFormat(8, 7)
FP16 = FloatFormat(5, 10)
E4M3 = FloatFormat(4, 3)
E5M2 = FloatFormat(5, 2)
_NAMED = {"fp32": FP32, "bf16": BF16, "fp16": FP16, "e4m3": E4M3, "e5m2": E5M2}


def parse_format(name: str) -> FloatFormat:
    """formats.py:148-156."""
    key = name.strip().lower()
    if key in _NAMED:
        return _NAMED[key]
    m = re.fullmatch(r"e(\d+)m(\d+)", key)
    if m is None:
        raise ValueError(f"unknown float format {name!r}")
    return FloatFormat(int(m.group(1)), int(m.group(2)))


def _check_finite(x):  # formats.py:159-161
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite input to rounding operation")


def _ulp_of(fmt: FloatFormat, x):
    """Grid spacing at |x|'s binade, float64 exact.  formats.py:164-168."""
    _, e = np.frexp(x)
    exp = np.clip(e - 1, fmt.min_normal_exp, fmt.max_exp)
    return np.ldexp(1.0, exp - fmt.man_bits)


def _saturate(fmt: FloatFormat, q, x):  # formats.py:171-177
    over = np.abs(q) > fmt.max_finite
    if np.any(over):
        if not fmt.saturating:
            raise OverflowError("value outside representable range of non-saturating format")
        q = np.where(over, np.copysign(fmt.max_finite, x), q)
    return q


def neighbors(fmt: FloatFormat, x):
    """Bracketing grid values, saturating.  formats.py:180-194."""
    x = np.asarray(x, dtype=np.float64)
    _check_finite(x)
    ulp = _ulp_of(fmt, x)
    f = x / ulp
    lo = _saturate(fmt, np.floor(f) * ulp, x)
    hi = _saturate(fmt, np.ceil(f) * ulp, x)
    clipped = np.abs(x) > fmt.max_finite
    lo = np.where(clipped, np.copysign(fmt.max_finite, x), lo)
    hi = np.where(clipped, np.copysign(fmt.max_finite, x), hi)
    return np.float32(lo), np.float32(hi)


def round_nearest(fmt: FloatFormat, x):
    """RTN ties-to-even onto the grid, saturating.  formats.py:197-206."""
    scalar = np.isscalar(x) or (isinstance(x, np.ndarray) and x.ndim == 0)
    x = np.asarray(x, dtype=np.float64)
    _check_finite(x)
    ulp = _ulp_of(fmt, x)
    q = _saturate(fmt, np.round(x / ulp) * ulp, x)
    q32 = np.float32(q)
    return np.float32(q32) if scalar else q32


def round_stochastic(fmt: FloatFormat, x, rng, step, tensor_id, index):
    """SR: hi if u < (x-lo)/(hi-lo) else lo.  formats.py:209-225."""
    x = np.asarray(x, dtype=np.float64)
    lo, hi = neighbors(fmt, x)
    lo64 = lo.astype(np.float64)
    hi64 = hi.astype(np.float64)
    width = hi64 - lo64
    with np.errstate(invalid="ignore", divide="ignore"):
        p = np.where(width > 0.0, (x - lo64) / width, 0.0)
    u = np.broadcast_to(np.asarray(rng.uniform(step, tensor_id, index)), x.shape)
    return np.where(u < p, hi, lo).astype(np.float32)


def kahan_add(s, c, v, fmt: FloatFormat):
    """Compensated add onto the grid; returns (sum, comp).  formats.py:246-263."""
    v = np.asarray(v, dtype=np.float32)
    _check_finite(v)
    s = np.asarray(s, dtype=np.float32)
    c = np.asarray(c, dtype=np.float32)
    if fmt.is_working_precision:
        return s + v, c
    y = v - c
    t = round_nearest(fmt, s + y)
    return t, (t - s) - y


# ---------------------------------------------------------------------------
# rng.py restatement

_GAMMA = np.uint64(0x9E3779B97F4A7C15)   # rng.py:15-19
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_U64 = np.uint64
_INV_2_53 = 1.0 / (1 << 53)


def _mix(z):
    """splitmix64 finalizer.  rng.py:22-25."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U64(30))) * _M1
        z = (z ^ (z >> _U64(27))) * _M2
        return z ^ (z >> _U64(31))


def tensor_tag(name: str) -> int:
    """FNV-1a 64.  rng.py:28-33."""
    h = 0xCBF29CE484222325
    for b in name.encode("utf-8"):
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


class RoundingRng:
    """Keyed uniform draws.  rng.py:36-57."""

    def __init__(self, seed: int):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF

    def _base(self, step: int, tensor_id: int):  # rng.py:42-46
        with np.errstate(over="ignore"):
            h = _mix(_U64(self.seed) + _GAMMA)
            h = _mix(h + _U64(step & 0xFFFFFFFFFFFFFFFF) * _GAMMA)
            h = _mix(h + _U64(tensor_id & 0xFFFFFFFFFFFFFFFF) * _GAMMA)
        return h

    def base(self, step: int, tensor_id: int) -> int:
        return int(self._base(step, tensor_id))

    def bits(self, step, tensor_id, index):  # rng.py:48-52
        idx = np.asarray(index, dtype=np.uint64)
        with np.errstate(over="ignore"):
            return _mix(self._base(step, tensor_id) + idx * _GAMMA)

    def uniform(self, step, tensor_id, index):  # rng.py:54-57
        h = self.bits(step, tensor_id, index)
        return (h >> _U64(11)).astype(np.float64) * _INV_2_53


# ---------------------------------------------------------------------------
# optimizers.py restatement


@dataclass
class SgdSrConfig:
    """optimizers.py:28-41."""

    lr: float
    weight_decay: float = 0.0
    fmt: FloatFormat = field(default_factory=lambda: FP32)
    rounding: str = "stochastic"

    def __post_init__(self):
        if self.lr <= 0:
            raise ValueError("lr must be positive")
        if self.weight_decay < 0:
            raise ValueError("weight_decay must be non-negative")
        if self.rounding not in ("stochastic", "nearest"):
            raise ValueError(f"unknown rounding mode {self.rounding!r}")


def sgd_sr_values(w, grad, cfg: SgdSrConfig, rng, step, tensor_id, global_index):
    """w <- ROUND(w - lr*(grad + wd*w)); one rounding.  optimizers.py:51-74
    (with _round_update :44-48).  Returns the new float32 values."""
    w = np.asarray(w, dtype=np.float32)
    grad = np.asarray(grad, dtype=np.float32)
    if grad.shape != w.shape:
        raise ValueError(f"shape mismatch: weights {w.shape}, grad {grad.shape}")
    if not np.all(np.isfinite(grad)):
        raise ValueError("non-finite gradient entry")
    g = grad if cfg.weight_decay == 0.0 else grad + np.float32(cfg.weight_decay) * w
    updated = w - np.float32(cfg.lr) * g
    if cfg.rounding == "stochastic":
        return round_stochastic(cfg.fmt, updated, rng, step, tensor_id, global_index)
    return round_nearest(cfg.fmt, updated)


def kahan_sgd_values(w, comp, grad, cfg: SgdSrConfig, rng, step, tensor_id,
                     global_index, comp_fmt=None):
    """Head-Kahan extension composed from
    kahan_add (formats.py:246-263) and the SGD update (optimizers.py:51-74):
        v = -lr*(g + wd*s); y = v - c; t = ROUND(s + y); c = (t - s) - y.
    ROUND is RTN (exactly kahan_add) or SR keyed like sgd_sr_step.  The
    compensation is kept in float32 here; the GPU may store it in bf16.
    Returns (new_w, new_comp)."""
    s = np.asarray(w, dtype=np.float32)
    c = np.asarray(comp, dtype=np.float32)
    grad = np.asarray(grad, dtype=np.float32)
    if not np.all(np.isfinite(grad)):
        raise ValueError("non-finite gradient entry")
    g = grad if cfg.weight_decay == 0.0 else grad + np.float32(cfg.weight_decay) * s
    v = -(np.float32(cfg.lr) * g)
    if cfg.fmt.is_working_precision:
        return s + v, c
    y = v - c
    x = s + y
    if cfg.rounding == "stochastic":
        t = round_stochastic(cfg.fmt, x, rng, step, tensor_id, global_index)
    else:
        t = round_nearest(cfg.fmt, x)
    c_new = (t - s) - y
    if comp_fmt is not None:   # compensation stored on a grid (bf16 in the paper)
        c_new = round_nearest(comp_fmt, c_new)
    return t, c_new


@dataclass
class KahanAdamWConfig:
    """optimizers.py:77-91."""

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


def kahan_adamw_values(w, comp, m, v, grad, cfg: KahanAdamWConfig, t: int, lr=None):
    """AdamW with Kahan-compensated parameter accumulation, optimizers.py:112-137
    (moments in float32, bias-corrected; decoupled weight decay; kahan_add
    formats.py:246-263 onto cfg.fmt).  Returns (w, comp, m, v) as new arrays;
    the reference updates its KahanAdamWParam in place."""
    if t < 1:
        raise ValueError("step index t must be >= 1")
    grad = np.asarray(grad, dtype=np.float32)
    w = np.asarray(w, dtype=np.float32)
    if grad.shape != w.shape:
        raise ValueError("gradient shape mismatch")
    lr = np.float32(cfg.lr if lr is None else lr)
    b1, b2 = np.float32(cfg.beta1), np.float32(cfg.beta2)
    m = b1 * np.asarray(m, np.float32) + (np.float32(1) - b1) * grad
    v = b2 * np.asarray(v, np.float32) + (np.float32(1) - b2) * grad * grad
    if not np.all(np.isfinite(m)) or not np.all(np.isfinite(v)):
        raise ValueError("non-finite optimizer moments")
    mhat = m / np.float32(1.0 - cfg.beta1 ** t)
    vhat = v / np.float32(1.0 - cfg.beta2 ** t)
    update = -lr * (mhat / (np.sqrt(vhat) + np.float32(cfg.eps)) + np.float32(cfg.weight_decay) * w)
    s_new, c_new = kahan_add(w, comp, update, cfg.fmt)
    return s_new, c_new, m, v


# ---------------------------------------------------------------------------
# head.py restatement

N_CELLS = 64                                   # head.py:40
HEAD_WEIGHTS_TAG = tensor_tag("head.weights")  # head.py:42
DROPOUT_TAG = tensor_tag("head.dropout")       # head.py:43
SIG_LO = np.float32(2.0 ** -24)                # head.py:47-48
SIG_HI = np.float32(1.0) - np.float32(2.0 ** -24)


def partition(total: int, parts: int):
    """head.py:51-57."""
    if parts < 1:
        raise ValueError("need at least one part")
    b = [(i * total) // parts for i in range(parts + 1)]
    return [(b[i], b[i + 1]) for i in range(parts) if b[i + 1] > b[i]]


def canonical_pieces(start: int, stop: int, total: int):
    """head.py:60-66."""
    cuts = sorted({start, stop}
                  | {b for b, _ in partition(total, min(N_CELLS, max(total, 1)))
                     if start < b < stop})
    cuts = [c for c in cuts if start <= c <= stop]
    return [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]


@dataclass
class OracleHead:
    """State of ChunkedHead (head.py:69-112): on-grid float32 weights."""

    values: np.ndarray          # (L, d) float32 on fmt's grid
    fmt: FloatFormat
    num_chunks: int = 1
    dropout_p: float = 0.0
    block_m: int = 64
    block_n: int = 64
    tensor_id: int = HEAD_WEIGHTS_TAG

    @classmethod
    def create(cls, num_labels, dim, fmt, seed=0, num_chunks=1, dropout_p=0.0,
               init_scale=0.02):  # head.py:86-92
        w = np.random.default_rng(seed).normal(
            scale=init_scale, size=(num_labels, dim)).astype(np.float32)
        return cls(round_nearest(fmt, w), fmt, num_chunks, dropout_p)

    @property
    def num_labels(self):
        return self.values.shape[0]

    @property
    def dim(self):
        return self.values.shape[1]

    def chunks(self):  # head.py:106-107
        return partition(self.num_labels, self.num_chunks)

    def scores(self, X):  # head.py:109-112
        Xq = round_nearest(self.fmt, np.asarray(X, dtype=np.float32))
        return Xq @ self.values.T


def dropout_mask(rng, step, p, row_range, num_cols):
    """head.py:138-152."""
    if not (0.0 <= p < 1.0):
        raise ValueError("dropout probability must lie in [0, 1)")
    start, stop = row_range
    rows = np.arange(start, stop, dtype=np.uint64)[:, None]
    flat = rows * np.uint64(num_cols) + np.arange(num_cols, dtype=np.uint64)[None, :]
    return (rng.uniform(step, DROPOUT_TAG, flat) >= p).astype(np.float32)


def _effective_weights(head, start, stop, rng, step):  # head.py:155-161
    w = head.values[start:stop]
    if head.dropout_p == 0.0:
        return w
    mask = dropout_mask(rng, step, head.dropout_p, (start, stop), head.dim)
    return w * (mask / np.float32(1.0 - head.dropout_p))


def head_forward_logits(head, chunk, Xq, rng, step):
    """(chunk labels, batch) fp32 logits per canonical piece.  head.py:164-178."""
    start, stop = chunk
    if Xq.shape[1] != head.dim:
        raise ValueError(f"input dim {Xq.shape[1]} != head dim {head.dim}")
    out = np.empty((stop - start, Xq.shape[0]), dtype=np.float32)
    for s, e in canonical_pieces(start, stop, head.num_labels):
        out[s - start:e - start] = _effective_weights(head, s, e, rng, step) @ Xq.T
    return out


def logit_gradient(logits, sample_idx, label_idx, chunk):
    """clip(sigmoid(z)) - Y.  head.py:181-196."""
    start, stop = chunk
    label_idx = np.asarray(label_idx, dtype=np.int64)
    if label_idx.size and (label_idx.min() < start or label_idx.max() >= stop):
        raise ValueError(f"label outside chunk range [{start}, {stop})")
    with np.errstate(over="ignore"):
        g = np.clip(1.0 / (1.0 + np.exp(-logits.astype(np.float32))), SIG_LO, SIG_HI)
    g = g.astype(np.float32)
    g[label_idx - start, np.asarray(sample_idx, dtype=np.int64)] -= np.float32(1.0)
    return g


def input_gradient_accumulate(acc, G, head, chunk, rng, step):
    """acc += G^T @ W per canonical piece.  head.py:199-209."""
    start, stop = chunk
    if acc.shape != (G.shape[1], head.dim):
        raise ValueError("accumulator shape mismatch")
    for s, e in canonical_pieces(start, stop, head.num_labels):
        acc += G[s - start:e - start].T @ _effective_weights(head, s, e, rng, step)
    return acc


def fused_weight_update(head, G, Xq, cfg, rng, step, chunk, comp=None, comp_fmt=None, adam=None):
    """Per 64-row block: scratch = G_rows @ Xq, then the SGD+rounding step
    keyed by the global flat index.  head.py:212-251 (rounding vectorised
    across the row block; see module docstring).  With ``comp`` (float32
    (n, d) array) the head-Kahan extension kahan_sgd_values is used for rows
    < n (n = L: every row; n < L: top-p% head-Kahan, on
    frequency-sorted labels) and the plain SR step for the others.

    Adam-style head (north_star "SGD or Adam-style update"; no reference head
    oracle exists, so this is the composition): with a KahanAdamWConfig and
    ``adam = {"m": m, "v": v, "t": t, "lr": lr_or_None}`` (float32 (L, d)
    moments, ``comp`` float32 (L, d)) every block's scratch goes through
    kahan_adamw_values (optimizers.py:112-137) instead of the SGD step."""
    start, stop = chunk
    m = head.dim
    keep = np.float32(1.0 - head.dropout_p)
    for s, e in canonical_pieces(start, stop, head.num_labels):
        for r0 in range(s, e, head.block_m):
            r1 = min(r0 + head.block_m, e)
            scratch = G[r0 - start:r1 - start] @ Xq
            if not np.all(np.isfinite(scratch)):
                raise ValueError("non-finite values in fused scratch block")
            if head.dropout_p > 0.0:
                scratch = scratch * (dropout_mask(rng, step, head.dropout_p,
                                                  (r0, r1), m) / keep)
            if isinstance(cfg, KahanAdamWConfig):
                (head.values[r0:r1], comp[r0:r1], adam["m"][r0:r1], adam["v"][r0:r1]) = kahan_adamw_values(
                    head.values[r0:r1], comp[r0:r1], adam["m"][r0:r1], adam["v"][r0:r1], scratch, cfg,
                    adam["t"], adam.get("lr"))
                continue
            idx = (np.arange(r0, r1, dtype=np.uint64)[:, None] * np.uint64(m)
                   + np.arange(m, dtype=np.uint64)[None, :])
            n_c = 0 if comp is None else min(max(comp.shape[0] - r0, 0), r1 - r0)
            if n_c > 0:
                head.values[r0:r0 + n_c], comp[r0:r0 + n_c] = kahan_sgd_values(
                    head.values[r0:r0 + n_c], comp[r0:r0 + n_c], scratch[:n_c], cfg, rng, step,
                    head.tensor_id, idx[:n_c], comp_fmt)
            if n_c < r1 - r0:
                head.values[r0 + n_c:r1] = sgd_sr_values(head.values[r0 + n_c:r1], scratch[n_c:], cfg,
                                                         rng, step, head.tensor_id, idx[n_c:])


def quantize_g_operand(G, fmt, g_format="e5m2"):
    """The GPU's operand-precision mode (ChunkedHead(precision="operand"))
    consumes G in the backward tensor-core operand format: an e4m3 head uses
    e5m2(G * 2^8) * 2^-8 (g_format "e5m2", the default) or e4m3(G * 2^8) * 2^-8
    ("e4m3") -- exact power-of-two scale -- or bf16(G) ("bf16", the paper's
    BF16 logit gradients), and a bf16 head uses bf16(G); all
    RTN.  This is a documented B200 design choice (not in the reference), so
    parity tests of that mode can isolate it by applying it here.  The default
    reference-precision mode needs no quantisation (g_quant=False)."""
    G = np.asarray(G, dtype=np.float32)
    if fmt.name == "e4m3" and g_format == "bf16":
        return round_nearest(BF16, G)   # the paper's BF16 logit gradients, unscaled
    if fmt.name == "e4m3":
        q = E5M2 if g_format == "e5m2" else E4M3
        return (round_nearest(q, G * np.float32(256.0)) * np.float32(1.0 / 256.0)).astype(np.float32)
    return round_nearest(fmt, G)


def head_update(head, X, sample_idx, label_idx, cfg, rng, step, comp=None,
                probe=None, g_quant=False, comp_fmt=None, adam=None):
    """One head step over all chunks; returns grad_X (b, d).  head.py:254-298.
    ``g_quant`` ("e5m2" / "e4m3", or True = "e5m2") applies
    quantize_g_operand to each chunk's G before the backward (the GPU's
    operand-precision mode); False (default) is the reference itself."""
    X = np.asarray(X, dtype=np.float32)
    sample_idx = np.asarray(sample_idx, dtype=np.int64)
    label_idx = np.asarray(label_idx, dtype=np.int64)
    Xq = round_nearest(head.fmt, X)
    acc = np.zeros((X.shape[0], head.dim), dtype=np.float32)
    order = np.lexsort((label_idx, sample_idx))
    ss, sl = sample_idx[order], label_idx[order]
    for chunk in head.chunks():
        start, stop = chunk
        inc = (sl >= start) & (sl < stop)
        logits = head_forward_logits(head, chunk, Xq, rng, step)
        G = logit_gradient(logits, ss[inc], sl[inc], chunk)
        del logits
        if probe is not None:
            probe(step, chunk, G)
        if g_quant:
            G = quantize_g_operand(G, head.fmt, "e5m2" if g_quant is True else g_quant)
        input_gradient_accumulate(acc, G, head, chunk, rng, step)
        fused_weight_update(head, G, Xq, cfg, rng, step, chunk, comp, comp_fmt, adam)
    return acc


# ---------------------------------------------------------------------------
# metrics.py restatement (the P@k judge)


def top_k_indices(scores, k):
    """Stable descending order, ties to the lower index.  metrics.py:38-47."""
    scores = np.asarray(scores)
    if scores.size == 0:
        raise ValueError("empty score vector")
    if not (1 <= k <= scores.size):
        raise ValueError(f"k must lie in [1, {scores.size}]")
    return np.argsort(-scores, kind="stable")[:k]


def precision_at_k(scores, truth, k):  # metrics.py:50-54
    top = top_k_indices(scores, k)
    truth = set(int(t) for t in truth)
    return sum(1 for l in top if int(l) in truth) / k


def dataset_precision_at_k(score_matrix, truths, k):  # metrics.py:76-79
    return float(np.mean([precision_at_k(s, t, k)
                          for s, t in zip(score_matrix, truths)]))


# ---------------------------------------------------------------------------
# checkpoint payload (head.py:304-392)

_MAGIC = b"LPXH"


def encode_grid_bits(values, fmt):
    """On-grid float32 -> sign/exp/mantissa bits.  head.py:317-338."""
    v = np.asarray(values, dtype=np.float64)
    sign = (v < 0) | ((v == 0) & (np.copysign(1.0, v) < 0))
    mag = np.abs(v)
    mant, e = np.frexp(mag)
    exp = e - 1
    normal = mag >= np.ldexp(1.0, fmt.min_normal_exp)
    exp_field = np.where(normal, exp + fmt.bias, 0).astype(np.int64)
    frac = np.where(normal,
                    np.ldexp(mag, -(exp.astype(np.int64)) + fmt.man_bits) - (1 << fmt.man_bits),
                    np.ldexp(mag, -fmt.min_exp))
    frac_i = np.rint(frac).astype(np.int64)
    if not np.array_equal(frac_i.astype(np.float64), frac):
        raise ValueError("value not on the format grid")
    bits = (sign.astype(np.int64) << (fmt.exp_bits + fmt.man_bits)) \
        | (exp_field << fmt.man_bits) | frac_i
    dt = np.uint8 if fmt.storage_bits <= 8 else (np.uint16 if fmt.storage_bits <= 16 else np.uint32)
    return bits.astype(dt)


def decode_grid_bits(bits, fmt):
    """head.py:341-355."""
    b = np.asarray(bits).astype(np.int64)
    frac = b & ((1 << fmt.man_bits) - 1)
    exp_field = (b >> fmt.man_bits) & ((1 << fmt.exp_bits) - 1)
    sign = (b >> (fmt.exp_bits + fmt.man_bits)) & 1
    mag = np.where(exp_field > 0,
                   np.ldexp((1 << fmt.man_bits) + frac.astype(np.float64),
                            exp_field - fmt.bias - fmt.man_bits),
                   np.ldexp(frac.astype(np.float64), fmt.min_exp))
    return np.where(sign == 1, -mag, mag).astype(np.float32)


def checkpoint_bytes(values, fmt) -> bytes:
    """save_head byte stream.  head.py:358-372."""
    tag = fmt.name.encode("ascii")
    L, m = values.shape
    return (_MAGIC + struct.pack("<IQQB", 1, L, m, len(tag)) + tag
            + encode_grid_bits(values, fmt).tobytes())


# ---------------------------------------------------------------------------
# synthetic workload (data.py:179-188 semantics)


def synthetic_positives(num_labels, batch, mean_labels, seed=0):
    """Per sample n ~ max(1, Poisson(mean)) distinct labels drawn Zipf(1.0)
    over [0, L) without replacement; returns (sample_idx, label_idx) int64
    sorted by (sample, label)."""
    rng = np.random.default_rng(seed)
    ranks = np.arange(1, num_labels + 1, dtype=np.float64)
    p = 1.0 / ranks
    p /= p.sum()
    cdf = np.cumsum(p)
    rows, cols = [], []
    for i in range(batch):
        n = max(1, int(rng.poisson(mean_labels)))
        n = min(n, num_labels)
        chosen = set()
        while len(chosen) < n:
            draw = np.searchsorted(cdf, rng.random(2 * n), side="right")
            for lab in np.minimum(draw, num_labels - 1):
                if len(chosen) < n:
                    chosen.add(int(lab))
        for lab in sorted(chosen):
            rows.append(i)
            cols.append(lab)
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)
