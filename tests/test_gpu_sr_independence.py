"""Independence of the production stochastic-rounding decisions (SR_FAST:
keyed-hash or Philox4x32-7 words fed to the hardware cvt.rs conversion,
through the fused backward epilogue).  Unbiasedness and per-decile
calibration are in test_gpu_parity.py; here every weight of a head gets an
update value at the SAME fractional position p between its two grid
neighbours, so each weight's round-up indicator is a Bernoulli(p) draw, and
the Pearson correlation between the indicators of element pairs must be
within 4 sigma (sigma = 1/sqrt(pairs)) of zero for:

  * the lanes of one cvt.rs.e4m3x4 instruction that share a 16-bit field
    (elements 4i, 4i+1 and 4i+2, 4i+3; the hardware reads the field
    bit-reversed for one lane of each pair, profiles/r1_probe_cvt_rs.txt --
    exhaustively over the 2^16 fields the correlation is <= 4e-4 for the p
    tested here) and the lanes of different halves (4i, 4i+2);
  * bf16x2 lanes (2i, 2i+1) and elements 16 apart (the word ranges of
    neighbouring threads, c and c+16);
  * neighbouring words, thread boundaries (c = 32j+31, 32j+32), neighbouring
    rows, and the same element in consecutive steps (the key changes).
"""

import numpy as np
import pytest
import torch

from oracle import lpxmc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xmc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_11168_b200 as xmc
    return xmc


def _indicators(xmc, fname, impl, p, step, L=4096, d=256, B=128):
    """Round-up indicators U[r, c] of one fused update where every element's
    exact update value sits at fraction p between its grid neighbours."""
    fmt, ofmt = xmc.parse_format(fname), O.parse_format(fname)
    w0, lo, ulp = (0.3125, 0.28125, 2.0 ** -5) if fname == "e4m3" else (1.0078125, 1.0, 2.0 ** -7)
    # x = w0 - lr * g with g = 0.5: lr chosen so that x = lo + p * ulp
    lr = float(np.float32((w0 - lo - p * ulp) / 0.5))
    x = np.float64(np.float32(w0) - np.float32(lr) * np.float32(0.5))
    lo_, hi_ = O.neighbors(ofmt, x)
    W = np.full((L, d), w0, np.float32)
    X = np.zeros((B, d), np.float32)
    X[0, :] = 1.0
    G = np.zeros((L, B), np.float32)
    G[:, 0] = 0.5
    head = xmc.ChunkedHead.from_float(torch.from_numpy(W), fmt, precision="operand")
    cfg = xmc.SgdSrConfig(lr=lr, fmt=fmt, rounding="stochastic", sr_impl=impl)
    xmc.fused_weight_update(head, torch.from_numpy(G).cuda(), torch.from_numpy(X), cfg, xmc.RoundingRng(5), step,
                            (0, L))
    got = head.weights.values.float().cpu().numpy()
    assert set(np.unique(got)) <= {float(lo_), float(hi_)}
    return (got == hi_).astype(np.float64), float((x - lo_) / (hi_ - lo_))


def _corr_ok(a, b, what):
    a, b = a.ravel(), b.ravel()
    c = np.corrcoef(a, b)[0, 1]
    sigma = 1.0 / np.sqrt(a.size)
    assert abs(c) < 4 * sigma, (what, c, sigma)


@pytest.mark.parametrize("impl", ["hash", "philox"])
@pytest.mark.parametrize("p", [0.5, 0.3, 0.1])
def test_e4m3_sr_decisions_independent(xmc, impl, p):
    U, pe = _indicators(xmc, "e4m3", impl, p, step=1)
    assert abs(U.mean() - pe) < 4 * np.sqrt(pe * (1 - pe) / U.size)
    _corr_ok(U[:, 0::4], U[:, 1::4], "shared 16-bit field (d, c)")
    _corr_ok(U[:, 2::4], U[:, 3::4], "shared 16-bit field (b, a)")
    _corr_ok(U[:, 0::4], U[:, 2::4], "halves of one word")
    _corr_ok(U[:, 0:-4], U[:, 4:], "neighbouring words")
    _corr_ok(U[:, 31:-1:32], U[:, 32::32], "thread boundary")
    _corr_ok(U[:-1], U[1:], "neighbouring rows")
    U2, _ = _indicators(xmc, "e4m3", impl, p, step=2)
    _corr_ok(U, U2, "consecutive steps")


@pytest.mark.parametrize("impl", ["hash", "philox"])
@pytest.mark.parametrize("p", [0.5, 0.3, 0.1])
def test_bf16_sr_decisions_independent(xmc, impl, p):
    U, pe = _indicators(xmc, "bf16", impl, p, step=1)
    assert abs(U.mean() - pe) < 4 * np.sqrt(pe * (1 - pe) / U.size)
    _corr_ok(U[:, 0::2], U[:, 1::2], "bf16x2 lanes")
    _corr_ok(U[:, :-16], U[:, 16:], "elements 16 apart")
    _corr_ok(U[:, :-1], U[:, 1:], "neighbouring elements")
    _corr_ok(U[:, 31:-1:32], U[:, 32::32], "thread boundary")
    _corr_ok(U[:-1], U[1:], "neighbouring rows")
    U2, _ = _indicators(xmc, "bf16", impl, p, step=2)
    _corr_ok(U, U2, "consecutive steps")
