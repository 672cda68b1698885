"""The fast backward specialisations (e4m3 head; keyed-hash SR or RTN; plain or
head-Kahan with the bf16 compensation staged by TMA with the W tile,
PAPER.md:795, formats.py:246-263 composed with optimizers.py:51-74) against
the general instantiation of the same kernel (XMC_BWD_GENERAL=1) on the same
inputs and keys: the two compute the same fp32 operations in the same order
and draw the same SR words, so weights and compensation must agree bit for
bit -- no / full / top-p % compensation (prefix ending inside a tile), one
and two chunks.  The general path itself is pinned to the oracle in
test_gpu_parity.py / test_gpu_reference.py."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2510_11168_b200 as xmc
from oracle import lpxmc_oracle as O
L, d, B, k, kl, out, rmode = int(sys.argv[2]), 768, 256, int(sys.argv[3]), int(sys.argv[4]), sys.argv[5], sys.argv[6]
rs = np.random.default_rng(3)
W = O.round_nearest(O.E4M3, rs.normal(scale=0.02, size=(L, d)).astype(np.float32))
f = xmc.parse_format("e4m3")
head = xmc.ChunkedHead.from_float(torch.from_numpy(W), f, num_chunks=k, precision="operand",
                                  kahan=("bf16" if kl >= 0 else None), kahan_labels=(kl if kl > 0 else None))
cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=f, rounding=rmode, sr_impl="hash")
for step in range(3):
    X = rs.normal(size=(B, d)).astype(np.float32)
    si, li = O.synthetic_positives(L, B, 5.0, seed=10 + step)
    gx = xmc.head_update(head, xmc.BatchInput(X, si, li), cfg, xmc.RoundingRng(5), step)
torch.cuda.synchronize()
c = head.comp.view(torch.int16).cpu().numpy() if head.comp is not None else np.zeros(1, np.int16)
np.savez(out, w=head.weights.values.view(torch.uint8).cpu().numpy(), c=c, gx=gx.cpu().numpy())
"""


def _run(tmp_path, L, k, kl, general, rmode):
    out = str(tmp_path / f"r_{L}_{k}_{kl}_{rmode}_{int(general)}.npz")
    env = dict(os.environ)
    if general:
        env["XMC_BWD_GENERAL"] = "1"
    else:
        env.pop("XMC_BWD_GENERAL", None)
    subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(L), str(k), str(kl), out, rmode], env=env, check=True,
                   timeout=600)
    return np.load(out)


@pytest.mark.parametrize("rmode", ["stochastic", "nearest"])
@pytest.mark.parametrize("L,k,kl", [(3000, 1, 0), (3000, 2, 0), (5000, 2, 1000), (5000, 1, 70), (3000, 2, -1)])
def test_fast_backward_equals_general(tmp_path, L, k, kl, rmode):
    """kl: compensated labels (0 = all, -1 = no head-Kahan)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _run(tmp_path, L, k, kl, general=False, rmode=rmode)
    b = _run(tmp_path, L, k, kl, general=True, rmode=rmode)
    assert np.array_equal(a["w"], b["w"]), int((a["w"] != b["w"]).sum())
    assert np.array_equal(a["c"], b["c"]), int((a["c"] != b["c"]).sum())
    np.testing.assert_allclose(a["gx"], b["gx"], rtol=1e-6, atol=1e-6)
    if kl >= 0:   # the compensation is live (not all zero) inside the prefix
        assert np.any(a["c"] != 0)
