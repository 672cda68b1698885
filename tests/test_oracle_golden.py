"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  Integer/byte work is checked bit-exact;
GEMM-derived values within fp32 tolerance."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import lpxmc_oracle as O  # noqa: E402

GOLD = np.load(os.path.join(ROOT, "tests", "golden", "lpxmc_golden.npz"))
NCASES = int(GOLD["head_ncases"])


def _bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def test_tensor_tags():
    for name, tag in zip(GOLD["rng_tag_names"], GOLD["rng_tags"]):
        assert O.tensor_tag(str(name)) == int(tag)
    assert O.HEAD_WEIGHTS_TAG == 0xfc05a0526df64580


def test_rng_bits_and_uniform_bit_exact():
    idx = GOLD["rng_idx"]
    for (seed, step, tag), bits, uni in zip(GOLD["rng_keys"], GOLD["rng_bits"],
                                            GOLD["rng_uniform"]):
        r = O.RoundingRng(int(seed))
        assert np.array_equal(r.bits(int(step), int(tag), idx), bits)
        assert np.array_equal(r.uniform(int(step), int(tag), idx).view(np.uint64),
                              uni.view(np.uint64))


@pytest.mark.parametrize("name", ["bf16", "e4m3", "e5m2", "fp16", "e3m2", "e2m1"])
def test_rounding_bit_exact(name):
    fmt = O.parse_format(name)
    x = GOLD["fmt_inputs"]
    assert O.FloatFormat.max_finite.fget(fmt) == float(GOLD[f"maxfinite_{name}"])
    assert np.array_equal(_bits(O.round_nearest(fmt, x)), _bits(GOLD[f"rtn_{name}"]))
    lo, hi = O.neighbors(fmt, x)
    assert np.array_equal(_bits(lo), _bits(GOLD[f"lo_{name}"]))
    assert np.array_equal(_bits(hi), _bits(GOLD[f"hi_{name}"]))
    sr = O.round_stochastic(fmt, x, O.RoundingRng(42), 5, O.HEAD_WEIGHTS_TAG, GOLD["sr_idx"])
    assert np.array_equal(_bits(sr), _bits(GOLD[f"sr_{name}"]))


def test_rounding_known_answers():
    # test_formats.py:26-52, 124-140 style KATs
    assert O.E4M3.max_finite == 448.0 and O.E5M2.max_finite == 57344.0
    assert (O.E4M3.min_exp, O.E4M3.max_exp) == (-9, 8)
    assert O.round_nearest(O.E4M3, 17.0) == 16.0 and O.round_nearest(O.E4M3, 19.0) == 20.0
    assert O.round_nearest(O.E4M3, 1e9) == 448.0
    assert np.signbit(O.round_nearest(O.E4M3, -1e-30))


def test_sr_many_keys_unbiased_and_matches():
    got = O.round_stochastic(O.E4M3, np.full(4096, np.float32(0.3)), O.RoundingRng(42),
                             9, 77, np.arange(4096, dtype=np.uint64))
    assert np.array_equal(_bits(got), _bits(GOLD["sr_many_e4m3"]))
    lo, hi = 0.28125, 0.3125
    p = (0.3 - lo) / (hi - lo)
    frac_hi = np.mean(got == np.float32(hi))
    assert abs(frac_hi - p) < 4 * np.sqrt(p * (1 - p) / 4096)


def test_kahan_known_answer():
    s = O.round_nearest(O.BF16, np.array([1.0, 256.0, -3.0, 0.5], np.float32))
    c = np.zeros(4, np.float32)
    for _ in range(4096):
        s, c = O.kahan_add(s, c, np.full(4, 2.0**-12, np.float32), O.BF16)
    assert np.array_equal(_bits(s), _bits(GOLD["kahan_sum"]))
    assert np.array_equal(_bits(c), _bits(GOLD["kahan_comp"]))
    assert s[0] == 2.0  # test_formats.py:216-229: 1 + 4096*2^-12 == 2 with Kahan


@pytest.mark.parametrize("name", ["bf16", "e4m3"])
@pytest.mark.parametrize("rmode", ["nearest", "stochastic"])
def test_sgd_step_bit_exact(name, rmode):
    fmt = O.parse_format(name)
    cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding=rmode)
    got = O.sgd_sr_values(GOLD[f"sgd_{name}_w"], GOLD[f"sgd_{name}_grad"], cfg,
                          O.RoundingRng(3), 4, O.HEAD_WEIGHTS_TAG, GOLD[f"sgd_{name}_idx"])
    assert np.array_equal(_bits(got), _bits(GOLD[f"sgd_{name}_{rmode}"]))


def test_partition_and_pieces():
    for total, k, a, b in GOLD["partition"]:
        assert (a, b) in O.partition(int(total), int(k))
    for total, k, a, b, s, e in GOLD["pieces"]:
        assert (s, e) in O.canonical_pieces(int(a), int(b), int(total))


@pytest.mark.parametrize("ci", range(NCASES))
def test_head_update_matches_reference(ci):
    p = f"head{ci}_"
    L, d, b, k = (int(v) for v in GOLD[p + "meta"])
    lr, wd, drop, seed = GOLD[p + "cfg"]
    fmt = O.parse_format(str(GOLD[p + "fmt"]))
    cfg = O.SgdSrConfig(lr=float(lr), weight_decay=float(wd), fmt=fmt,
                        rounding=str(GOLD[p + "rounding"]))
    head = O.OracleHead(GOLD[p + "W0"].copy(), fmt, k, float(drop))
    rng = O.RoundingRng(int(seed))
    X, si, li = GOLD[p + "X"], GOLD[p + "sample_idx"], GOLD[p + "label_idx"]
    Xq = O.round_nearest(fmt, X)
    c0 = head.chunks()[0]
    logits = O.head_forward_logits(head, c0, Xq, rng, 0)
    np.testing.assert_allclose(logits, GOLD[p + "logits0"], rtol=1e-5, atol=1e-5)
    inc = (li >= c0[0]) & (li < c0[1])
    G = O.logit_gradient(logits, si[inc], li[inc], c0)
    np.testing.assert_allclose(G, GOLD[p + "G0"], rtol=1e-5, atol=1e-6)
    for step, (gx_key, w_key) in enumerate([("gradX1", "W1"), ("gradX2", "W2")]):
        gx = O.head_update(head, X, si, li, cfg, rng, step)
        np.testing.assert_allclose(gx, GOLD[p + gx_key], rtol=1e-4, atol=1e-4)
        # weights: within one grid ulp everywhere, almost all bit-identical
        ref = GOLD[p + w_key]
        diff = head.values != ref
        assert diff.mean() < 0.01
        if diff.any():
            lo, hi = O.neighbors(fmt, ref[diff].astype(np.float64))
            ulp = np.maximum(np.abs(hi - lo), O._ulp_of(fmt, ref[diff]))
            assert np.all(np.abs(head.values[diff] - ref[diff]) <= 2 * ulp + 1e-30)
        head.values = ref.copy()  # re-sync so step 2 is checked independently
    ck = O.checkpoint_bytes(head.values, fmt)
    assert ck == GOLD[p + "ckpt"].tobytes()


def test_topk_and_precision():
    sc = GOLD["topk_scores"]
    for s, ref in zip(sc, GOLD["topk_5"]):
        assert np.array_equal(O.top_k_indices(s, 5), ref)
    flat, lens = GOLD["topk_truth_flat"], GOLD["topk_truth_len"]
    truths = np.split(flat, np.cumsum(lens)[:-1])
    got = [O.dataset_precision_at_k(sc, truths, k) for k in (1, 3, 5)]
    assert np.allclose(got, GOLD["p_at_k"], rtol=0, atol=0)


def test_grid_bits_roundtrip():
    for name in ["bf16", "e4m3", "e5m2"]:
        fmt = O.parse_format(name)
        v = O.round_nearest(fmt, np.random.default_rng(1).normal(size=1000).astype(np.float32))
        assert np.array_equal(_bits(O.decode_grid_bits(O.encode_grid_bits(v, fmt), fmt)), _bits(v))


@pytest.mark.parametrize("name", ["bf16", "e4m3", "fp32"])
def test_kahan_adamw_bit_exact(name):
    """kahan_adamw_step (optimizers.py:112-137) over four steps, lr override on
    steps 2 and 4: parameter, compensation and both moments bit-exact."""
    fmt = O.parse_format(name)
    cfg = O.KahanAdamWConfig(lr=0.01, beta1=0.9, beta2=0.99, eps=1e-6, weight_decay=0.05, fmt=fmt)
    w = GOLD[f"adamw_{name}_w0"]
    c = np.zeros_like(w)
    m = np.zeros_like(w)
    v = np.zeros_like(w)
    for t, (g, lr) in enumerate(zip(GOLD[f"adamw_{name}_grads"], GOLD[f"adamw_{name}_lrs"]), start=1):
        w, c, m, v = O.kahan_adamw_values(w, c, m, v, g, cfg, t, lr=None if np.isnan(lr) else float(lr))
        for arr, key in ((w, "w"), (c, "c"), (m, "m"), (v, "v")):
            assert np.array_equal(_bits(arr), _bits(GOLD[f"adamw_{name}_{key}{t}"])), (key, t)


def test_kahan_adamw_config_validation():
    with pytest.raises(ValueError):
        O.KahanAdamWConfig(lr=0.1, beta1=1.0)
    with pytest.raises(ValueError):
        O.KahanAdamWConfig(lr=0.1, eps=0.0)
    with pytest.raises(ValueError):
        O.kahan_adamw_values(np.zeros(2, np.float32), np.zeros(2, np.float32), np.zeros(2, np.float32),
                             np.zeros(2, np.float32), np.zeros(2, np.float32), O.KahanAdamWConfig(lr=0.1), 0)
