"""Chunked extreme-classification head on B200 -- mirror of lpxmc.head.

Same names, argument meaning and errors as the reference module
(/root/reference/pkg/src/lpxmc/head.py), on torch CUDA tensors:

* ``ChunkedHead.weights.values`` is the NATIVE weight tensor (torch.bfloat16
  or torch.float8_e4m3fn, L x d, row-major); its bytes equal the reference's
  ``encode_grid_bits`` payload (head.py:317-338).  No fp32 master copy.
* ``head_update`` (head.py:254-298) runs the whole step in two tcgen05
  kernels per chunk through the C ABI (include/xmc_head.h):
  logits+G (head.py:164-196) then grad_X + dW + SGD/rounding (head.py:199-251).
* ``ChunkedHead.precision`` selects the precision of G in the two backward
  GEMMs.  ``"reference"`` (default): G is the reference's fp32 logit gradient,
  split exactly into three bf16 planes, so dW and grad_X multiply by the same
  fp32 G as the reference (head.py:193-208, 236) and only the fp32
  accumulation order differs.  ``"operand"``: the production fast path, G
  rounded once to the FP8/BF16 tensor-core operand format (e4m3 heads:
  ``g_format`` "e5m2" (default, e5m2(2^8 g): the reference's whole
  [2^-24, 1] sigmoid range), "e4m3" (e4m3(2^8 g)) or "bf16" (bf16(g): the
  paper's FP8 weights with BF16 logit gradients -- the e4m3 W tiles become
  bf16 operands in shared memory, kind::f16 backward GEMMs, batch <= 256);
  bf16 heads: bf16(g)).
* The unfused sub-ops keep the reference signatures for parity isolation.

There is no CPU fallback: every call goes to libxmc_b200.so.
"""

from __future__ import annotations

from dataclasses import dataclass
import ctypes
import io
import struct

import numpy as np
import torch

from . import _lib
from .formats import FloatFormat, RoundingRng, parse_format, tensor_tag
from .optimizers import KahanAdamWConfig, SgdSrConfig

__all__ = [
    "ChunkedHead", "BatchInput", "QuantizedMatrix", "partition", "canonical_pieces",
    "head_forward_logits", "logit_gradient", "input_gradient_accumulate",
    "fused_weight_update", "head_update", "save_head", "load_head",
    "HEAD_WEIGHTS_TAG", "DROPOUT_TAG", "N_CELLS",
]

N_CELLS = 64                                   # head.py:40
HEAD_WEIGHTS_TAG = tensor_tag("head.weights")  # head.py:42
DROPOUT_TAG = tensor_tag("head.dropout")       # head.py:43


def partition(total: int, parts: int) -> list[tuple[int, int]]:
    """head.py:51-57."""
    if parts < 1:
        raise ValueError("need at least one part")
    b = [(i * total) // parts for i in range(parts + 1)]
    return [(b[i], b[i + 1]) for i in range(parts) if b[i + 1] > b[i]]


def canonical_pieces(start: int, stop: int, total: int) -> list[tuple[int, int]]:
    """head.py:60-66 (kept for API parity; the GPU kernels are per-row
    deterministic, so results do not depend on piece boundaries)."""
    cuts = sorted({start, stop} | {b for b, _ in partition(total, min(N_CELLS, max(total, 1)))
                                   if start < b < stop})
    cuts = [c for c in cuts if start <= c <= stop]
    return [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]


@dataclass
class QuantizedMatrix:
    """Weights in native storage (formats.py:306-327 with native bytes)."""

    values: torch.Tensor
    fmt: FloatFormat

    @property
    def shape(self):
        return tuple(self.values.shape)

    def float(self) -> torch.Tensor:
        return self.values.float()


class _Handle:
    """C-ABI head handle plus its torch-owned device workspace."""

    def __init__(self, head: "ChunkedHead", max_batch: int, max_positives: int):
        lib = _lib.load()
        self.key = (max_batch, max_positives, head.num_chunks, head.weights.values.device)
        comp_bytes = 0 if head.comp is None else head.comp.element_size()
        self.precision, self.g_format = head.precision, head.g_format
        self.desc = _lib.HeadDesc(head.num_labels_global, head.label_offset, head.num_labels,
                                  head.dim, head.fmt.code, head.num_chunks, max_batch,
                                  max_positives, 0, comp_bytes, 1 if head.dropout_p > 0.0 else 0,
                                  _PRECISIONS[head.precision], head.kahan_labels or 0,
                                  _G_FORMATS[head.g_format], 0)
        size = ctypes.c_size_t()
        _lib.check(lib.xmc_head_workspace_size(ctypes.byref(self.desc), ctypes.byref(size)))
        self.workspace = torch.empty(size.value + 1024, dtype=torch.uint8,
                                     device=head.weights.values.device)
        base = (self.workspace.data_ptr() + 1023) // 1024 * 1024
        self.h = ctypes.c_void_p()
        _lib.check(lib.xmc_head_create(ctypes.byref(self.desc), base, size.value, ctypes.byref(self.h)))
        self.max_batch, self.max_positives = max_batch, max_positives

    def __del__(self):
        try:
            if self.h:
                _lib.load().xmc_head_destroy(self.h)
        except Exception:
            pass


_PRECISIONS = {"reference": _lib.PRECISION_REFERENCE, "operand": _lib.PRECISION_OPERAND}
_G_FORMATS = {"e5m2": _lib.FMT_E5M2, "e4m3": _lib.FMT_E4M3, "bf16": _lib.FMT_BF16}


class ChunkedHead:
    """Classifier weights partitioned into contiguous label chunks (head.py:69-112).

    ``num_labels_global`` / ``label_offset`` describe this rank's shard when
    the head is label-sharded across GPUs (see parallel.ShardedHead); for a
    single GPU they are (L, 0).  ``precision`` / ``g_format``: the backward's G
    precision (module docstring)."""

    def __init__(self, weights: QuantizedMatrix, num_chunks: int = 1, dropout_p: float = 0.0,
                 block_m: int = 64, block_n: int = 64, tensor_id: int = HEAD_WEIGHTS_TAG,
                 num_labels_global: int | None = None, label_offset: int = 0,
                 kahan: str | None = None, kahan_labels: int | None = None, adamw: bool = False,
                 precision: str = "reference", g_format: str = "e5m2"):
        if num_chunks < 1:
            raise ValueError("num_chunks must be >= 1")
        if not (0.0 <= dropout_p < 1.0):
            raise ValueError("dropout_p must lie in [0, 1)")
        if precision not in _PRECISIONS:
            raise ValueError(f"precision must be 'reference' or 'operand', got {precision!r}")
        if g_format not in _G_FORMATS:
            raise ValueError(f"g_format must be 'e5m2', 'e4m3' or 'bf16', got {g_format!r}")
        self.precision, self.g_format = precision, g_format
        if weights.values.dtype != weights.fmt.torch_dtype or weights.fmt.code not in (
                _lib.FMT_BF16, _lib.FMT_E4M3):
            raise NotImplementedError("GPU head stores bf16 or e4m3 weights natively")
        if not weights.values.is_cuda:
            raise ValueError("head weights must live on a CUDA device")
        self.weights = weights
        self.num_chunks = num_chunks
        self.dropout_p = dropout_p
        self.block_m, self.block_n = block_m, block_n
        self.tensor_id = tensor_id
        self.num_labels_global = num_labels_global or weights.values.shape[0]
        self.label_offset = label_offset
        # head-Kahan compensation buffer (PAPER.md:795 uses bf16)
        if kahan not in (None, "bf16", "fp32"):
            raise ValueError("kahan must be None, 'bf16' or 'fp32'")
        # top-p% head-Kahan: only GLOBAL labels < kahan_labels
        # (the most frequent ones, labels sorted by frequency) keep a
        # compensation; this shard's comp buffer holds its rows of that prefix
        self.kahan_labels = kahan_labels
        n_comp = weights.values.shape[0] if kahan_labels is None else max(
            0, min(weights.values.shape[0], kahan_labels - label_offset))
        # Adam-style head (head_update with a KahanAdamWConfig): fp32 moments
        # and an fp32 compensation for every label, as kahan_adamw_step keeps
        if adamw:
            if kahan not in (None, "fp32") or kahan_labels is not None:
                raise ValueError("the Adam-style head keeps an fp32 compensation for every label")
            kahan, n_comp = "fp32", weights.values.shape[0]
        self.comp = None if kahan is None else torch.zeros(
            (n_comp, weights.values.shape[1]), dtype=torch.bfloat16 if kahan == "bf16" else torch.float32,
            device=weights.values.device)
        self.adam_m = torch.zeros_like(self.comp) if adamw else None
        self.adam_v = torch.zeros_like(self.comp) if adamw else None
        self._handle = None
        self.last_stats = None
        self.collect_stats = False   # True: head_update also returns sum|G| in last_stats[0]
        self.peers = None            # parallel.PeerGroup: head_update returns the node's summed grad_X

    # -- construction -------------------------------------------------------
    @classmethod
    def create(cls, num_labels: int, dim: int, fmt: FloatFormat, seed: int = 0,
               num_chunks: int = 1, dropout_p: float = 0.0, init_scale: float = 0.02,
               device="cuda", **kw) -> "ChunkedHead":
        """Same W0 as the reference (head.py:86-92): numpy N(0, scale^2) then
        RTN onto the grid -- the RTN cast runs on the GPU, bit-exact."""
        w = np.random.default_rng(seed).normal(scale=init_scale, size=(num_labels, dim)).astype(np.float32)
        return cls(QuantizedMatrix(cast_native(torch.from_numpy(w).to(device), fmt), fmt),
                   num_chunks, dropout_p, **kw)

    @classmethod
    def from_float(cls, values, fmt: FloatFormat, **kw) -> "ChunkedHead":
        """Wrap on-grid float values (e.g. a reference QuantizedMatrix.values)."""
        t = torch.as_tensor(np.asarray(values, dtype=np.float32) if not isinstance(values, torch.Tensor)
                            else values, dtype=torch.float32)
        return cls(QuantizedMatrix(cast_native(t.to(kw.pop("device", "cuda")), fmt), fmt), **kw)

    # -- reference properties -------------------------------------------------
    @property
    def num_labels(self) -> int:
        return self.weights.values.shape[0]

    @property
    def dim(self) -> int:
        return self.weights.values.shape[1]

    @property
    def fmt(self) -> FloatFormat:
        return self.weights.fmt

    def chunks(self) -> list[tuple[int, int]]:
        return partition(self.num_labels, self.num_chunks)

    def scores(self, X) -> torch.Tensor:
        """Inference logits (batch, L_local) fp32 (head.py:109-112)."""
        X = _as_x(X, self.dim)
        out = torch.empty((self.num_labels, X.shape[0]), dtype=torch.float32, device=X.device)
        h = self.handle(X.shape[0], 0)
        _lib.check(_lib.load().xmc_head_logits(h.h, self.weights.values.data_ptr(), X.data_ptr(),
                                               X.shape[0], 0, self.num_labels, out.data_ptr(),
                                               X.shape[0], None, _lib.stream_ptr()))
        return out.t()

    def topk(self, X, k: int) -> tuple[torch.Tensor, torch.Tensor]:
        """Per-sample top-k of ``scores(X)`` without materialising it: (scores
        (B, k) fp32, GLOBAL labels (B, k) int64), ordered like
        metrics.top_k_indices (metrics.py:38-47: descending, ties toward the
        lower label).  One fused tcgen05 launch + a per-sample merge; k <= 8."""
        X = _as_x(X, self.dim)
        b = X.shape[0]
        vals = torch.empty((b, k), dtype=torch.float32, device=X.device)
        labs = torch.empty((b, k), dtype=torch.int64, device=X.device)
        h = self.handle(b, 0)
        _lib.check(_lib.load().xmc_head_topk(h.h, self.weights.values.data_ptr(), X.data_ptr(), b, k,
                                             vals.data_ptr(), labs.data_ptr(), _lib.stream_ptr()))
        return vals, labs

    # -- plumbing -----------------------------------------------------------
    def handle(self, batch: int, nnz: int) -> _Handle:
        h = self._handle
        dev = self.weights.values.device
        comp_bytes = 0 if self.comp is None else self.comp.element_size()
        if (h is None or batch > h.max_batch or nnz > h.max_positives
                or h.key[2] != self.num_chunks or h.key[3] != dev or h.desc.comp_bytes != comp_bytes
                or h.desc.dropout != (1 if self.dropout_p > 0.0 else 0)
                or h.precision != self.precision or h.g_format != self.g_format):
            mb = max(batch, h.max_batch if h else 0)
            mp = max(nnz, h.max_positives if h else 0, 1024)
            self._handle = _Handle(self, mb, mp)
        return self._handle


@dataclass
class BatchInput:
    """Batch embeddings plus sparse positives as (sample, label) pairs (head.py:115-135)."""

    X: object
    sample_idx: object
    label_idx: object

    @classmethod
    def from_label_lists(cls, X, labels) -> "BatchInput":
        rows = [i for i, ls in enumerate(labels) for _ in ls]
        cols = [l for ls in labels for l in ls]
        return cls(X, np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64))


def cast_native(x: torch.Tensor, fmt: FloatFormat) -> torch.Tensor:
    """RTN cast of float32 values onto fmt's grid in native storage (GPU kernel)."""
    x = x.to(torch.float32).contiguous()
    out = torch.empty(x.shape, dtype=fmt.torch_dtype, device=x.device)
    st = torch.zeros(1, dtype=torch.int32, device=x.device)
    _lib.check(_lib.load().xmc_cast_rn(x.data_ptr(), out.data_ptr(), x.numel(), fmt.code,
                                       st.data_ptr(), _lib.stream_ptr()))
    if int(st.item()) != 0:
        raise ValueError("non-finite input to rounding operation")
    return out


def dropout_mask(rng: RoundingRng, step: int, p: float, row_range: tuple[int, int],
                 num_cols: int, device="cuda") -> torch.Tensor:
    """Keep/drop mask (rows x num_cols) float32 of a global row slice
    (head.py:138-152), generated on the GPU bit-exactly (integer threshold on
    the splitmix64 draw)."""
    if not (0.0 <= p < 1.0):
        raise ValueError("dropout probability must lie in [0, 1)")
    start, stop = row_range
    wpr = (num_cols + 31) // 32
    words = torch.empty((max(stop - start, 0), wpr), dtype=torch.int32, device=device)
    _lib.check(_lib.load().xmc_dropout_mask(start, stop, num_cols, rng.seed, step & (2**64 - 1), float(p),
                                            words.data_ptr(), _lib.stream_ptr()))
    bits = torch.arange(32, dtype=torch.int32, device=device)
    m = (words.unsqueeze(-1) >> bits) & 1
    return m.reshape(words.shape[0], wpr * 32)[:, :num_cols].to(torch.float32)


def _as_x(X, dim) -> torch.Tensor:
    t = torch.as_tensor(X, dtype=torch.float32) if not isinstance(X, torch.Tensor) else X.to(torch.float32)
    if not t.is_cuda:
        t = t.cuda(non_blocking=True)
    t = t.contiguous()
    if t.dim() != 2 or t.shape[1] != dim:
        raise ValueError(f"input dim {t.shape[-1]} != head dim {dim}")
    return t


def _as_idx(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a.to(torch.int32)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64).astype(np.int32)))
    return t.to(device, non_blocking=True).contiguous().reshape(-1)


def _step_args(cfg: SgdSrConfig | None, rng: RoundingRng, step: int, tensor_id: int,
               dropout_p: float = 0.0) -> _lib.StepArgs:
    lr, wd, rc = (cfg.lr, cfg.weight_decay, cfg.rounding_code) if cfg is not None else (0.0, 0.0, 0)
    bits = cfg.sr_bits if cfg is not None else 0
    return _lib.StepArgs(lr, wd, rc, bits, rng.seed, step & (2**64 - 1), tensor_id & (2**64 - 1),
                         float(dropout_p))


def _dropout_args(head: "ChunkedHead", rng: RoundingRng, step: int):
    """Step args carrying only the dropout key (seed, step, p), or None at p = 0."""
    if head.dropout_p == 0.0:
        return None
    return ctypes.byref(_step_args(None, rng, step, head.tensor_id, head.dropout_p))


def _check_cfg(head: ChunkedHead, cfg: SgdSrConfig):
    if cfg.fmt != head.fmt:
        raise ValueError(f"SgdSrConfig.fmt {cfg.fmt.name} != head format {head.fmt.name}; "
                         "the head stores weights natively in its own grid")


# --------------------------------------------------------------- hot path

def head_update(head: ChunkedHead, batch: BatchInput, cfg: SgdSrConfig, rng: RoundingRng,
                step: int, tracker=None, probe=None, check: bool = True,
                grad_out: torch.Tensor | None = None) -> torch.Tensor:
    """One full head step over all chunks; returns grad_X (b, d) fp32 on the
    device (head.py:254-298).  W is updated in place.  ``check`` synchronises
    and raises device-detected errors like the reference (non-finite X or
    gradient -> ValueError, bad sample index -> IndexError)."""
    _check_cfg(head, cfg)
    if isinstance(cfg, KahanAdamWConfig) and head.adam_m is None:
        raise ValueError("head_update with a KahanAdamWConfig needs ChunkedHead(..., adamw=True)")
    dev = head.weights.values.device
    X = _as_x(batch.X, head.dim)
    si = _as_idx(batch.sample_idx, dev)
    li = _as_idx(batch.label_idx, dev)
    if si.numel() != li.numel():
        raise ValueError("sample_idx and label_idx differ in length")
    b = X.shape[0]
    acc_h = None
    if tracker is not None:  # same tags/sizes as the reference (head.py:267-283)
        acc_h = tracker.alloc("input_grad_accumulator", "accumulator", b * head.dim * 4)
    try:
        if probe is not None:
            if head.peers is not None:
                raise NotImplementedError("probe + peer all-reduce: use the fused step (probe=None)")
            if head.comp is not None:
                raise NotImplementedError("probe + head-Kahan: use the fused step (probe=None)")
            return _head_update_unfused(head, X, si, li, cfg, rng, step, tracker, probe)
        h = head.handle(b, si.numel())
        # node-local peer all-reduce of grad_X (parallel.PeerGroup), or none
        _lib.check(_lib.load().xmc_head_attach_peers(h.h, head.peers.p if head.peers is not None else None))
        gx = grad_out if grad_out is not None else torch.empty((b, head.dim), dtype=torch.float32, device=dev)
        stats_ptr = None
        if head.collect_stats:  # sum |G| of the step (trainer divergence proxy)
            if head.last_stats is None or head.last_stats.device != dev:
                head.last_stats = torch.zeros(2, dtype=torch.float32, device=dev)
            stats_ptr = head.last_stats.data_ptr()
        lhs = []
        if tracker is not None:
            for s, e in head.chunks():
                lhs.append(tracker.alloc("chunk_logits", "logits", (e - s) * b * 2))
        if isinstance(cfg, KahanAdamWConfig):
            # Adam-style head: t = step + 1 (head_update steps are 0-based)
            args = _step_args(None, rng, step, head.tensor_id, head.dropout_p)
            adam = _lib.AdamWArgs(cfg.lr, cfg.weight_decay, cfg.eps, 0.0, cfg.beta1, cfg.beta2, step + 1)
            _lib.check(_lib.load().xmc_head_step_adamw(
                h.h, head.weights.values.data_ptr(), head.comp.data_ptr(), head.adam_m.data_ptr(),
                head.adam_v.data_ptr(), X.data_ptr(), b, si.data_ptr(), li.data_ptr(), si.numel(),
                ctypes.byref(adam), ctypes.byref(args), gx.data_ptr(), stats_ptr, _lib.stream_ptr()))
        else:
            args = _step_args(cfg, rng, step, head.tensor_id, head.dropout_p)
            _lib.check(_lib.load().xmc_head_step_kahan(
                h.h, head.weights.values.data_ptr(), _lib.ptr(head.comp), X.data_ptr(), b, si.data_ptr(),
                li.data_ptr(), si.numel(), ctypes.byref(args), gx.data_ptr(), stats_ptr, _lib.stream_ptr()))
        for lh in lhs:
            tracker.free(lh)
        if check:
            _lib.check(_lib.load().xmc_head_check(h.h, _lib.stream_ptr()))
        return gx
    finally:
        if acc_h is not None:
            tracker.free(acc_h)


def _head_update_unfused(head, X, si, li, cfg, rng, step, tracker, probe):
    acc = torch.zeros((X.shape[0], head.dim), dtype=torch.float32, device=X.device)
    for chunk in head.chunks():
        start, stop = chunk
        sel = (li >= start) & (li < stop)
        logits = head_forward_logits(head, chunk, X, rng, step)
        G = logit_gradient(logits, si[sel], li[sel], chunk)
        del logits
        probe(step, chunk, G)
        input_gradient_accumulate(acc, G, head, chunk, rng, step)
        fused_weight_update(head, G, X, cfg, rng, step, chunk, tracker)
    return acc


def head_forward_logits(head: ChunkedHead, chunk, Xq, rng, step) -> torch.Tensor:
    """Logits of one chunk, (chunk labels, batch) fp32 (head.py:164-178);
    W_eff = W * keep / (1 - p) under keyed dropout (head.py:155-161)."""
    start, stop = chunk
    X = _as_x(Xq, head.dim)
    out = torch.empty((stop - start, X.shape[0]), dtype=torch.float32, device=X.device)
    h = head.handle(X.shape[0], 0)
    _lib.check(_lib.load().xmc_head_logits(h.h, head.weights.values.data_ptr(), X.data_ptr(),
                                           X.shape[0], start, stop, out.data_ptr(), X.shape[0],
                                           _dropout_args(head, rng, step), _lib.stream_ptr()))
    return out


def logit_gradient(logits: torch.Tensor, sample_idx, label_idx, chunk) -> torch.Tensor:
    """sigmoid(logit) (clipped) at negatives, minus 1 at positives (head.py:181-196)."""
    start, stop = chunk
    z = logits.to(torch.float32).contiguous()
    if z.dim() != 2 or z.shape[0] != stop - start:
        raise ValueError("logits shape does not match chunk")
    si = _as_idx(sample_idx, z.device)
    li = _as_idx(label_idx, z.device)
    G = torch.empty_like(z)
    _lib.check(_lib.load().xmc_logit_gradient(z.data_ptr(), z.shape[0], z.shape[1], z.shape[1],
                                              si.data_ptr(), li.data_ptr(), si.numel(), start,
                                              G.data_ptr(), _lib.stream_ptr()))
    return G


def input_gradient_accumulate(acc: torch.Tensor, G: torch.Tensor, head: ChunkedHead, chunk,
                              rng, step) -> torch.Tensor:
    """acc += G^T @ W_chunk (head.py:199-209).  G is consumed at the head's
    backward precision (exact three-plane bf16 split by default)."""
    start, stop = chunk
    if tuple(acc.shape) != (G.shape[1], head.dim):
        raise ValueError("accumulator shape mismatch")
    Gc = G.to(torch.float32).contiguous()
    h = head.handle(G.shape[1], 0)
    _lib.check(_lib.load().xmc_head_backward(
        h.h, head.weights.values.data_ptr(), Gc.data_ptr(), Gc.shape[1], None, Gc.shape[1],
        start, stop, acc.data_ptr(), 1, 0, _dropout_args(head, rng, step), _lib.stream_ptr()))
    _lib.check(_lib.load().xmc_head_check(h.h, _lib.stream_ptr()))
    return acc


def fused_weight_update(head: ChunkedHead, G: torch.Tensor, Xq, cfg: SgdSrConfig, rng, step: int,
                        chunk, tracker=None) -> None:
    """Gradient + SGD + rounding per tile, in place, no resident gradient
    (head.py:212-251)."""
    _check_cfg(head, cfg)
    start, stop = chunk
    X = _as_x(Xq, head.dim)
    Gc = G.to(torch.float32).contiguous()
    h = head.handle(X.shape[0], 0)
    handle = None
    if tracker is not None:
        handle = tracker.alloc("fused_block_scratch", "scratch", head.block_m * head.block_n * 4)
    try:
        args = _step_args(cfg, rng, step, head.tensor_id, head.dropout_p)
        _lib.check(_lib.load().xmc_head_backward(
            h.h, head.weights.values.data_ptr(), Gc.data_ptr(), Gc.shape[1], X.data_ptr(),
            X.shape[0], start, stop, None, 0, 1, ctypes.byref(args), _lib.stream_ptr()))
        _lib.check(_lib.load().xmc_head_check(h.h, _lib.stream_ptr()))
    finally:
        if handle is not None:
            tracker.free(handle)


# --------------------------------------------------------------- checkpoint
_MAGIC = b"LPXH"
_VERSION = 1


def save_head(head: ChunkedHead, fp) -> None:
    """head.py:358-372: header + row-major grid bits.  The payload is the raw
    native bytes (identical to encode_grid_bits for bf16/e4m3)."""
    close = isinstance(fp, (str, bytes))
    if close:
        fp = open(fp, "wb")
    try:
        tag = head.fmt.name.encode("ascii")
        fp.write(_MAGIC)
        fp.write(struct.pack("<IQQB", _VERSION, head.num_labels, head.dim, len(tag)))
        fp.write(tag)
        raw = head.weights.values.contiguous().view(torch.uint8 if head.fmt.storage_bits <= 8
                                                    else torch.int16).cpu().numpy()
        fp.write(raw.tobytes())
    finally:
        if close:
            fp.close()


def load_head(fp, num_chunks: int = 1, dropout_p: float = 0.0, device="cuda", **kw) -> ChunkedHead:
    """head.py:375-392."""
    close = isinstance(fp, (str, bytes))
    if close:
        fp = open(fp, "rb")
    try:
        if fp.read(4) != _MAGIC:
            raise ValueError("not a head checkpoint (bad magic)")
        version, L, m, taglen = struct.unpack("<IQQB", fp.read(21))
        if version != _VERSION:
            raise ValueError(f"unsupported checkpoint version {version}")
        fmt = parse_format(fp.read(taglen).decode("ascii"))
        nbytes = 1 if fmt.storage_bits <= 8 else 2
        raw = np.frombuffer(fp.read(L * m * nbytes), dtype=np.uint8 if nbytes == 1 else np.int16)
        if raw.size != L * m:
            raise ValueError("truncated head checkpoint")
        t = torch.from_numpy(raw.copy()).reshape(L, m).to(device).view(fmt.torch_dtype)
        return ChunkedHead(QuantizedMatrix(t, fmt), num_chunks, dropout_p, **kw)
    finally:
        if close:
            fp.close()
