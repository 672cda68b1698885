"""Memory discipline of the head step (north_star: "never materialises a full
gradient buffer"; the reference's own check, /root/reference/pkg/tests/
test_head.py:335-347, only inspects a Python attribute).

Measured with the CUDA caching allocator's peak counter around head_update:

* steady state (handle and workspace exist): a step allocates no more than
  its small per-step tensors (the grad_X result, positives / X staging) --
  far below one chunk's fp32 gradient L_c * d * 4;
* the workspace itself is the chunk's G buffer (L_c x Bp operand bytes, or
  the three bf16 planes in reference precision) plus O(B d) and O(tiles)
  side buffers: it never reaches L_c * d * 4, and it shrinks with the chunk
  count.
"""

import numpy as np
import pytest
import torch

from oracle import lpxmc_oracle as O

pytestmark = pytest.mark.gpu

L, D, B = 400_000, 768, 256


@pytest.fixture(scope="module")
def xmc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11168_b200 as x
    return x


def _inputs():
    rs = np.random.default_rng(1)
    X = torch.from_numpy(rs.normal(size=(B, D)).astype(np.float32)).cuda()
    si, li = O.synthetic_positives(L, B, 36.17, seed=2)
    return X, torch.from_numpy(si.astype(np.int32)).cuda(), torch.from_numpy(li.astype(np.int32)).cuda()


@pytest.mark.parametrize("precision", ["operand", "reference"])
@pytest.mark.parametrize("k", [2, 4])
def test_step_allocates_no_gradient_buffer(xmc, precision, k):
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    W = xmc.cast_native(torch.randn((L, D), generator=g, device="cuda") * 0.02, xmc.E4M3)
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, xmc.E4M3), num_chunks=k, precision=precision)
    X, si, li = _inputs()
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=xmc.E4M3, rounding="stochastic")
    rng = xmc.RoundingRng(0)
    out = torch.empty((B, D), dtype=torch.float32, device="cuda")
    Lc = -(-L // k)
    full_grad = Lc * D * 4

    torch.cuda.synchronize()
    base0 = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, rng, 0, grad_out=out)
    torch.cuda.synchronize()
    first = torch.cuda.max_memory_allocated() - base0
    ws = head._handle.workspace.numel()
    # the first call creates the workspace; nothing else of chunk size
    assert first <= ws + (8 << 20), (first, ws)
    assert ws < full_grad, f"workspace {ws / 2**20:.1f} MiB >= one chunk's fp32 gradient {full_grad / 2**20:.1f} MiB"
    g_bytes = Lc * 256 * (6 if precision == "reference" else 1)
    assert ws <= g_bytes + (48 << 20), (ws, g_bytes)

    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    for s in range(1, 3):
        xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, rng, s, grad_out=out)
    torch.cuda.synchronize()
    steady = torch.cuda.max_memory_allocated() - base
    assert steady <= (4 << 20), f"a steady-state step allocated {steady / 2**20:.2f} MiB"
    print(f"{precision} k={k}: workspace {ws / 2**20:.1f} MiB (G {g_bytes / 2**20:.1f} MiB), "
          f"chunk fp32 gradient would be {full_grad / 2**20:.1f} MiB, steady-state step +{steady / 2**20:.2f} MiB")
