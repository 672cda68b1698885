"""Label-sharded head across GPUs.

One process per GPU.  Rank r owns the contiguous label rows
``partition(L, world)[r]`` (head.py:51-57) of W; a batch (X, positives with
GLOBAL label ids) is given to every rank, each rank runs the fused head step
on its shard (labels outside the shard are ignored there, exactly as the
reference ignores labels outside a chunk) and the partial input gradients are
summed with one all-reduce.  RNG keys use the global row index, so the
weights each rank ends with are the rows the single-GPU run would produce.

Evaluation (F1): per-rank scores -> per-rank top-k (score, global label) ->
all-gather -> merge with ties broken toward the lower label index, the
reference's ``top_k_indices`` order (metrics.py:38-47).
"""

from __future__ import annotations

import ctypes
from typing import Callable

import torch
import torch.distributed as dist

from . import _lib
from .head import ChunkedHead, partition


def shard_bounds(num_labels: int, world: int, rank: int) -> tuple[int, int]:
    """Rows owned by `rank` (head.py:51-57 partition)."""
    parts = partition(num_labels, world)
    if len(parts) != world:
        raise ValueError(f"cannot shard {num_labels} labels over {world} ranks")
    return parts[rank]


def topk_stable(scores: torch.Tensor, k: int, offset: int = 0) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-row top-k of a (B, L) score matrix with ties toward the lower index
    (metrics.py:38-47); returns (values, global indices)."""
    if not (1 <= k <= scores.shape[1]):
        raise ValueError(f"k must lie in [1, {scores.shape[1]}]")
    vals, idx = torch.topk(scores, k, dim=1, largest=True, sorted=True)
    kth = vals[:, -1:]
    n_ge = (scores >= kth).sum(dim=1)
    tied = (n_ge > k).nonzero().flatten()
    for r in tied.tolist():   # exact stable order only where the k-th score is tied
        order = torch.sort(-scores[r], stable=True).indices[:k]
        idx[r] = order
        vals[r] = scores[r, order]
    return vals, idx + offset


def merge_topk(vals: torch.Tensor, idx: torch.Tensor, k: int) -> torch.Tensor:
    """Merge per-rank candidates (B, world*k): order by (-score, label)."""
    # lexicographic key: sort by label first, then stable by -score
    o1 = torch.argsort(idx, dim=1, stable=True)
    v1, i1 = torch.gather(vals, 1, o1), torch.gather(idx, 1, o1)
    o2 = torch.argsort(-v1, dim=1, stable=True)
    return torch.gather(i1, 1, o2)[:, :k]


def broadcast_batch(X, sample_idx, label_idx, src: int = 0, group=None, out=None):
    """X broadcast of SURVEY.md 8(e): rank `src` holds the batch (encoder output
    X, B x d float32, and the positives as GLOBAL label ids); every other rank
    receives it.  Returns (X, sample_idx, label_idx) tensors on every rank, on
    the device of the process group's backend (CUDA for NCCL).

    ``out=(X, sample_idx, label_idx)``: preallocated receive tensors (float32,
    int32, int32) whose shapes every rank already knows, e.g. a training loop
    with a fixed batch and positive count: rank `src` copies its batch into
    them (host -> device when the inputs are pinned host tensors) and the
    shape exchange is skipped."""
    rank = dist.get_rank(group)
    if out is not None:
        Xo, so, lo_ = out
        if rank == src:
            Xo.copy_(torch.as_tensor(X), non_blocking=True)
            so.copy_(torch.as_tensor(sample_idx), non_blocking=True)
            lo_.copy_(torch.as_tensor(label_idx), non_blocking=True)
        dist.broadcast(Xo, src, group=group)
        if so.numel():
            dist.broadcast(so, src, group=group)
            dist.broadcast(lo_, src, group=group)
        return Xo, so, lo_
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    if rank == src:
        X = torch.as_tensor(X, dtype=torch.float32).to(dev).contiguous()
        si = torch.as_tensor(sample_idx, dtype=torch.int32).to(dev).contiguous()
        li = torch.as_tensor(label_idx, dtype=torch.int32).to(dev).contiguous()
        meta = torch.tensor([X.shape[0], X.shape[1], si.numel()], dtype=torch.int64, device=dev)
    else:
        meta = torch.empty(3, dtype=torch.int64, device=dev)
    dist.broadcast(meta, src, group=group)
    b, d, nnz = (int(v) for v in meta.tolist())
    if rank != src:
        X = torch.empty((b, d), dtype=torch.float32, device=dev)
        si = torch.empty(nnz, dtype=torch.int32, device=dev)
        li = torch.empty(nnz, dtype=torch.int32, device=dev)
    dist.broadcast(X, src, group=group)
    if nnz:
        dist.broadcast(si, src, group=group)
        dist.broadcast(li, src, group=group)
    return X, si, li


class PeerGroup:
    """Node-local grad_X all-reduce over peer memory (include/xmc_head.h,
    xmc_peer_*): replaces ``dist.all_reduce(grad_X)`` after the step.  Each
    rank allocates an exchange buffer, the CUDA IPC handles are swapped with
    one ``all_gather_object`` on ``group`` (any backend), and every peer buffer
    is mapped over NVLink.  Attached to a ChunkedHead, head_update's own
    grad_X reduction pushes each 32x32 tile to every rank and sums the ranks'
    tiles in rank order: one kernel, bit-identical grad_X on every rank.
    Raises RuntimeError when a peer buffer cannot be mapped (callers fall back
    to dist.all_reduce)."""

    def __init__(self, dim: int, max_batch: int, group=None):
        # Collective-safe: every rank takes part in both exchanges even when its
        # own step failed, and all ranks raise together, so no rank is left
        # waiting in a collective the others skipped.
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        lib = _lib.load()
        self.p = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        err = None
        try:
            _lib.check(lib.xmc_peer_create(self.rank, self.world, dim, max_batch, ctypes.byref(self.p),
                                           ctypes.cast(handle, ctypes.c_void_p)))
            mine = bytes(handle)
        except Exception as e:  # noqa: BLE001 - reported after the exchange
            err, mine = e, b""
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=group)
        if err is None and all(len(h) == 64 for h in handles):
            buf = (ctypes.c_char * (64 * self.world)).from_buffer_copy(b"".join(handles))
            try:
                _lib.check(lib.xmc_peer_connect(self.p, ctypes.cast(buf, ctypes.c_void_p)))
            except Exception as e:  # noqa: BLE001
                err = e
        elif err is None:
            err = RuntimeError("a peer rank could not create its exchange buffer")
        oks = [None] * self.world
        dist.all_gather_object(oks, err is None, group=group)
        if not all(oks):
            self.close()
            raise RuntimeError(f"peer group unavailable: {err or 'failed on another rank'}")

    def attach(self, head: ChunkedHead) -> None:
        head.peers = self

    def close(self) -> None:
        if self.p:
            _lib.load().xmc_peer_destroy(self.p)
            self.p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedHead:
    """A rank's shard of a label-sharded head.

    ``local_step(batch, cfg, rng, step) -> grad_X partial`` defaults to the
    fused GPU step on this rank's ChunkedHead; tests may inject another
    per-rank implementation to exercise the sharding logic on CPU (gloo).
    """

    def __init__(self, num_labels: int, rank: int, world: int, local: ChunkedHead | None = None,
                 group=None, local_step: Callable | None = None, local_scores: Callable | None = None):
        self.num_labels = num_labels
        self.rank, self.world = rank, world
        self.lo, self.hi = shard_bounds(num_labels, world, rank)
        self.local = local
        self.group = group
        if local is not None:
            if local.num_labels != self.hi - self.lo or local.label_offset != self.lo:
                raise ValueError("local head does not match this rank's shard")
        self._step = local_step or self._gpu_step
        self._fused_scores = local_scores is None
        self._scores = local_scores or (lambda X: self.local.scores(X))

    def _gpu_step(self, batch, cfg, rng, step):
        from .head import head_update
        return head_update(self.local, batch, cfg, rng, step)

    def head_update(self, batch, cfg, rng, step: int) -> torch.Tensor:
        """head_update over all shards; returns the full grad_X on every rank."""
        gx = self._step(batch, cfg, rng, step)
        if self.world > 1 and (self.local is None or self.local.peers is None):
            dist.all_reduce(gx, op=dist.ReduceOp.SUM, group=self.group)
        return gx

    def topk(self, X, k: int) -> torch.Tensor:
        """Global top-k label ids per sample (B, k).  A GPU shard ranks with the
        fused streaming top-k (no B x L_r score matrix); injected CPU scorers
        (gloo tests) go through topk_stable on their score matrix."""
        if self.local is not None and k <= 8 and self._scores is not None and self._fused_scores:
            vals, idx = self.local.topk(X, min(k, self.hi - self.lo))
        else:
            sc = self._scores(X)
            vals, idx = topk_stable(sc, min(k, sc.shape[1]), offset=self.lo)
        if self.world > 1:
            # gloo gathers host tensors only (the one-GPU test harness)
            dev = vals.device
            if dist.get_backend(self.group) != "nccl":
                vals, idx = vals.cpu(), idx.cpu()
            vs = [torch.empty_like(vals) for _ in range(self.world)]
            ix = [torch.empty_like(idx) for _ in range(self.world)]
            dist.all_gather(vs, vals.contiguous(), group=self.group)
            dist.all_gather(ix, idx.contiguous(), group=self.group)
            vals, idx = torch.cat(vs, dim=1).to(dev), torch.cat(ix, dim=1).to(dev)
        return merge_topk(vals, idx, k)
