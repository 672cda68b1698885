"""Label-sharded head on CPU with gloo, world_size 2.

The per-rank compute is the oracle (the GPU kernels need a device); what is
tested here is the host-side sharding: shard bounds, global-label filtering,
global-row RNG keys, the grad_X all-reduce and the top-k merge with the
reference's tie order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lpxmc_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rs = np.random.default_rng(3)
    L, d, B = 301, 32, 8
    W = O.round_nearest(O.BF16, rs.normal(scale=0.05, size=(L, d)).astype(np.float32))
    X = rs.normal(size=(B, d)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, 4.0, seed=4)
    return L, W, X, si, li


def _oracle_shard_step(W_shard, lo, hi, num_labels_global, k):
    """Per-rank step: oracle head on rows [lo, hi) keyed by GLOBAL rows."""
    head = O.OracleHead(W_shard, O.BF16, k)

    def step(batch, cfg, rng, step_i):
        X, si, li = batch
        keep = (li >= lo) & (li < hi)
        # run the oracle on the shard with global flat keys: emulate by an
        # oracle head over [0, hi) whose first lo rows are padding
        pad = O.OracleHead(np.zeros((hi, head.dim), np.float32), O.BF16, 1)
        pad.values[lo:hi] = head.values
        acc = np.zeros((X.shape[0], head.dim), np.float32)
        Xq = O.round_nearest(O.BF16, X)
        chunk = (lo, hi)
        logits = O.head_forward_logits(pad, chunk, Xq, rng, step_i)
        G = O.logit_gradient(logits, si[keep], li[keep], chunk)
        O.input_gradient_accumulate(acc, G, pad, chunk, rng, step_i)
        O.fused_weight_update(pad, G, Xq, cfg, rng, step_i, chunk)
        head.values[:] = pad.values[lo:hi]
        return torch.from_numpy(acc)

    return head, step


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_11168_b200.parallel import ShardedHead, shard_bounds
    L, W, X, si, li = _problem()
    lo, hi = shard_bounds(L, world, rank)
    head, step = _oracle_shard_step(W[lo:hi].copy(), lo, hi, L, 1)
    sh = ShardedHead(L, rank, world, local=None, local_step=step,
                     local_scores=lambda Xs: torch.from_numpy(head.scores(Xs)))
    cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=O.BF16, rounding="stochastic")
    gx = sh.head_update((X, si, li), cfg, O.RoundingRng(11), 0)
    top = sh.topk(X, 5)
    out[rank] = (gx.numpy(), head.values.copy(), top.numpy(), (lo, hi))
    dist.destroy_process_group()


def _bcast_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_11168_b200.parallel import broadcast_batch
    L, W, X, si, li = _problem()
    if rank == 0:
        Xb, sib, lib = broadcast_batch(X, si, li)
    else:
        Xb, sib, lib = broadcast_batch(None, None, None)
    # preallocated receive buffers (fixed batch shape): no shape exchange
    bufs = (torch.empty(X.shape, dtype=torch.float32), torch.empty(len(si), dtype=torch.int32),
            torch.empty(len(li), dtype=torch.int32))
    src = (torch.from_numpy(X), torch.from_numpy(si.astype(np.int32)), torch.from_numpy(li.astype(np.int32)))
    Xo, sio, lio = broadcast_batch(*(src if rank == 1 else (None, None, None)), src=1, out=bufs)
    assert Xo is bufs[0]
    out[rank] = (Xb.numpy(), sib.numpy(), lib.numpy(), Xo.numpy(), sio.numpy(), lio.numpy())
    dist.destroy_process_group()


def test_broadcast_batch():
    """X (and the global positives) broadcast from rank 0."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bcast_worker, args=(world, port, out), nprocs=world, join=True)
    L, W, X, si, li = _problem()
    for r in range(world):
        Xb, sib, lib, Xo, sio, lio = out[r]
        assert np.array_equal(Xb, X) and np.array_equal(sib, si) and np.array_equal(lib, li)
        assert np.array_equal(Xo, X) and np.array_equal(sio, si) and np.array_equal(lio, li)


def test_sharded_step_matches_single_process():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    L, W, X, si, li = _problem()
    full = O.OracleHead(W.copy(), O.BF16, 1)
    cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=O.BF16, rounding="stochastic")
    gx_ref = O.head_update(full, X, si, li, cfg, O.RoundingRng(11), 0)
    for r in range(world):
        gx, Wr, top, (lo, hi) = out[r]
        np.testing.assert_allclose(gx, gx_ref, rtol=1e-5, atol=1e-5)
        # global-row keys: each shard's weights equal the full run's rows
        diff = Wr != full.values[lo:hi]
        assert diff.mean() < 0.005
        ref_top = np.stack([O.top_k_indices(s, 5) for s in O.OracleHead(full.values, O.BF16).scores(X)])
        assert np.array_equal(top, ref_top)


def test_topk_merge_tie_order():
    from paper_2510_11168_b200.parallel import merge_topk, topk_stable
    sc = torch.tensor([[1.0, 3.0, 3.0, 0.5, 3.0, 2.0]])
    v, i = topk_stable(sc, 2)
    assert i.tolist() == [[1, 2]]
    # two "ranks" holding labels [0,3) and [3,6)
    va, ia = topk_stable(sc[:, :3], 2, offset=0)
    vb, ib = topk_stable(sc[:, 3:], 2, offset=3)
    m = merge_topk(torch.cat([va, vb], 1), torch.cat([ia, ib], 1), 3)
    assert m.tolist() == [list(O.top_k_indices(sc[0].numpy(), 3))]
