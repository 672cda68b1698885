"""Ranking metrics on the GPU (lpxmc.metrics, metrics.py:38-79).

``top_k_indices`` / ``precision_at_k`` / ``dataset_precision_at_k`` keep the
reference signatures on a materialised score matrix (stable descending order,
ties toward the lower label index).  ``head_precision_at_k`` is the streaming
path: the fused top-k kernel ranks every label of the head without
forming the B x L score matrix.
"""

from __future__ import annotations

import numpy as np
import torch


def top_k_indices(scores, k: int) -> torch.Tensor:
    """Indices of the k highest scores, ties broken by lower label index."""
    s = torch.as_tensor(scores)
    if s.numel() == 0:
        raise ValueError("empty score vector")
    if not (1 <= k <= s.numel()):
        raise ValueError(f"k must lie in [1, {s.numel()}]")
    return torch.sort(-s.reshape(-1), stable=True).indices[:k]


def precision_at_k(scores, truth, k: int) -> float:
    """|top_k(scores) intersect truth| / k."""
    top = top_k_indices(scores, k).tolist()
    t = set(int(x) for x in truth)
    return sum(1 for l in top if l in t) / k


def dataset_precision_at_k(score_matrix, truths: list, k: int) -> float:
    """Mean per-sample P@k."""
    return float(np.mean([precision_at_k(s, t, k) for s, t in zip(score_matrix, truths)]))


def precision_at_k_from_topk(top_labels, truths: list, k: int) -> float:
    """Mean P@k from per-sample ranked label lists (B, >= k)."""
    top = torch.as_tensor(top_labels)[:, :k].tolist()
    return float(np.mean([sum(1 for l in row if l in set(int(x) for x in t)) / k
                          for row, t in zip(top, truths)]))


def head_precision_at_k(head, X, truths: list, ks=(1, 3, 5)) -> dict:
    """Trainer.evaluate (trainer.py:245-250) on the streaming top-k path."""
    kmax = max(k for k in ks if k <= head.num_labels)
    _, labels = head.topk(X, kmax)
    return {f"p_at_{k}": precision_at_k_from_topk(labels, truths, k) for k in ks if k <= head.num_labels}
