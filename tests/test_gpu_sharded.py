"""parallel.ShardedHead with the real GPU step on every rank,
in the one-GPU harness: the rank processes share cuda:0 (gloo for the
host-side collectives, the peer all-reduce through CUDA IPC as over NVLink).

Per rank: the batch arrives by broadcast_batch from rank 0 (the other ranks
pass None), ShardedHead.head_update runs the fused step on the rank's label
shard and sums grad_X across ranks -- through the peer group, or through
dist.all_reduce when no peer group is attached -- and ShardedHead.topk merges
the per-rank fused top-k lists.  Checked against ONE process holding all
labels (same W0, batch, keys):

* every rank's weight rows are bit-identical to the single-process rows
  (global-row RNG keys), over several steps;
* grad_X equals the single-process grad_X within fp32 summation order, and
  is bitwise identical on every rank;
* the merged top-k equals the single-process fused top-k (ties toward the
  lower label).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

L, D, B, STEPS = 30_011, 768, 256, 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(xmc, fmt):
    from oracle import lpxmc_oracle as O
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    W0 = xmc.cast_native(torch.randn((L, D), generator=g, device="cuda") * 0.02, fmt)
    rs = np.random.default_rng(2)
    X = rs.normal(size=(B, D)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, 5.0, seed=3)
    return W0, X, si, li


def _worker(rank, world, port, fmt_name, peer, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2510_11168_b200 as xmc
    from paper_2510_11168_b200.parallel import PeerGroup, ShardedHead, broadcast_batch, shard_bounds
    fmt = xmc.parse_format(fmt_name)
    W0, X, si, li = _problem(xmc, fmt)
    lo, hi = shard_bounds(L, world, rank)
    local = xmc.ChunkedHead(xmc.QuantizedMatrix(W0[lo:hi].clone(), fmt), num_chunks=2, num_labels_global=L,
                            label_offset=lo, precision="operand")
    sh = ShardedHead(L, rank, world, local=local)
    pg = None
    if peer:
        pg = PeerGroup(D, B)
        pg.attach(local)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic")
    gxs = []
    for step in range(STEPS):
        # rank 0 holds the batch (encoder output + global positives)
        Xb, sib, lib = broadcast_batch(X, si, li) if rank == 0 else broadcast_batch(None, None, None)
        gx = sh.head_update(xmc.BatchInput(Xb.cuda(), sib.cuda(), lib.cuda()), cfg, xmc.RoundingRng(5), step)
        gxs.append(gx.cpu())
    top = sh.topk(torch.from_numpy(X).cuda(), 5).cpu()
    torch.cuda.synchronize()
    torch.save({"gx": gxs, "W": local.weights.values.view(torch.uint8).cpu(), "top": top, "lo": lo, "hi": hi},
               os.path.join(out_dir, f"rank{rank}.pt"))
    dist.barrier()
    if pg is not None:
        pg.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("fmt_name,world,peer", [("e4m3", 2, True), ("e4m3", 3, False), ("bf16", 2, True), ("e4m3", 4, True)])
def test_sharded_gpu_step_matches_single_process(tmp_path, fmt_name, world, peer):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mp.spawn(_worker, args=(world, _free_port(), fmt_name, peer, str(tmp_path)), nprocs=world, join=True)
    import paper_2510_11168_b200 as xmc
    fmt = xmc.parse_format(fmt_name)
    W0, X, si, li = _problem(xmc, fmt)
    full = xmc.ChunkedHead(xmc.QuantizedMatrix(W0.clone(), fmt), num_chunks=2, precision="operand")
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic")
    gx_ref = [xmc.head_update(full, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(5), s).cpu()
              for s in range(STEPS)]
    top_ref = full.topk(torch.from_numpy(X).cuda(), 5)[1].cpu()
    Wf = full.weights.values.view(torch.uint8).cpu()
    r = [torch.load(os.path.join(tmp_path, f"rank{k}.pt")) for k in range(world)]
    for k in range(world):
        assert torch.equal(r[k]["W"], Wf[r[k]["lo"]:r[k]["hi"]]), f"rank {k} weights differ from the full run"
        for s in range(STEPS):
            torch.testing.assert_close(r[k]["gx"][s], gx_ref[s], rtol=1e-5, atol=1e-4)
            assert torch.equal(r[k]["gx"][s], r[0]["gx"][s])
        assert torch.equal(r[k]["top"], top_ref)
