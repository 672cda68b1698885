"""Peer-memory grad_X all-reduce (parallel.PeerGroup, xmc_peer_* in
include/xmc_head.h) with two and three ranks.  The round's GPU box has one
B200, so the rank processes share cuda:0: the exchange buffers are still mapped through CUDA
IPC in the other process and every push / flag / wait runs as it does over
NVLink.  Per step and rank the peer result must equal the sum of the ranks'
partial grad_X from heads without peers (fp32 tolerance), be bitwise
identical on every rank, and leave each shard's weights bitwise equal to the
peer-less run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

L, D, B, STEPS = 40_000, 768, 256, 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fmt_name, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2510_11168_b200 as xmc
    from paper_2510_11168_b200.parallel import PeerGroup
    from oracle import lpxmc_oracle as O
    fmt = xmc.parse_format(fmt_name)
    lo, hi = xmc.partition(L, world)[rank]
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    W0 = xmc.cast_native(torch.randn((L, D), generator=g, device="cuda") * 0.02, fmt)[lo:hi].contiguous()
    rs = np.random.default_rng(2)
    X = rs.normal(size=(B, D)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, 5.0, seed=3)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding="stochastic")

    def make():
        return xmc.ChunkedHead(xmc.QuantizedMatrix(W0.clone(), fmt), num_chunks=2, num_labels_global=L,
                               label_offset=lo)

    plain, peered = make(), make()
    pg = PeerGroup(D, B)
    pg.attach(peered)
    res = {"expect": [], "got": []}
    for step in range(STEPS):
        part = xmc.head_update(plain, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(5), step).cpu()
        parts = [torch.empty_like(part) for _ in range(world)]
        dist.all_gather(parts, part)
        res["expect"].append(sum(parts[1:], parts[0].clone()))
        res["got"].append(xmc.head_update(peered, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(5), step).cpu())
    res["w_equal"] = bool(torch.equal(plain.weights.values.view(torch.uint8), peered.weights.values.view(torch.uint8)))
    torch.cuda.synchronize()
    torch.save(res, os.path.join(out_dir, f"rank{rank}.pt"))
    dist.barrier()
    pg.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("fmt_name,world", [("e4m3", 2), ("bf16", 2), ("e4m3", 3), ("e4m3", 8)])
def test_peer_allreduce_ranks(tmp_path, fmt_name, world):
    mp.spawn(_worker, args=(world, _free_port(), fmt_name, str(tmp_path)), nprocs=world, join=True)
    r = [torch.load(os.path.join(tmp_path, f"rank{k}.pt")) for k in range(world)]
    for k in range(world):
        assert r[k]["w_equal"]
        for step in range(STEPS):
            torch.testing.assert_close(r[k]["got"][step], r[k]["expect"][step], rtol=1e-5, atol=1e-5)
    for k in range(1, world):
        for step in range(STEPS):
            assert torch.equal(r[0]["got"][step], r[k]["got"][step])
