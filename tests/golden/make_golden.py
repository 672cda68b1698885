"""Generate golden vectors from the REFERENCE package (lpxmc) itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports ``lpxmc`` from /root/reference/pkg/src (read-only) and writes small
``.npz`` fixtures next to this file.  The fixtures are committed; nothing at
test time (CPU or GPU box) reads /root/reference.  Every vector below comes
from a reference call named in the comment (file:line of the reference).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    import lpxmc
    from lpxmc import formats as F, head as H, optimizers as O, rng as R, metrics as M

    out = {}

    # -- optimizers.py:112-137 kahan_adamw_step (+ kahan_add formats.py:246-263):
    # several steps on one parameter per format, with weight decay and an lr override
    rs = np.random.default_rng(99)
    for fname in ("bf16", "e4m3", "fp32"):
        fmt = F.parse_format(fname) if hasattr(F, "parse_format") else getattr(F, fname.upper())
        cfg = O.KahanAdamWConfig(lr=0.01, beta1=0.9, beta2=0.99, eps=1e-6, weight_decay=0.05, fmt=fmt)
        w0 = (rs.standard_normal(4096) * 0.3).astype(np.float32)
        param = O.KahanAdamWParam.from_values(w0, fmt)
        out[f"adamw_{fname}_w0"] = param.values.copy()
        grads = (rs.standard_normal((4, 4096)) * np.array([[1.0], [1e-3], [30.0], [1e-6]])).astype(np.float32)
        out[f"adamw_{fname}_grads"] = grads
        lrs = [None, 0.003, None, 0.02]
        out[f"adamw_{fname}_lrs"] = np.array([np.nan if x is None else x for x in lrs])
        for t, (g, lr) in enumerate(zip(grads, lrs), start=1):
            O.kahan_adamw_step(param, g, cfg, t, lr=lr)
            out[f"adamw_{fname}_w{t}"] = param.values.copy()
            out[f"adamw_{fname}_c{t}"] = param.state.comp.copy()
            out[f"adamw_{fname}_m{t}"] = param.m.copy()
            out[f"adamw_{fname}_v{t}"] = param.v.copy()

    # -- rng.py:22-57: tags, base keys, bits, uniforms ----------------------
    tags = ["head.weights", "head.dropout", "", "encoder.w1"]
    out["rng_tag_names"] = np.array(tags)
    out["rng_tags"] = np.array([R.tensor_tag(t) for t in tags], dtype=np.uint64)
    keys = [(0, 0, H.HEAD_WEIGHTS_TAG), (7, 3, H.HEAD_WEIGHTS_TAG),
            (2**63 + 5, 2**40, H.DROPOUT_TAG), (123456789, 1, 0)]
    idx = np.concatenate([np.arange(0, 64, dtype=np.uint64),
                          np.array([2**32 - 1, 2**32, 2**40 + 17, 2**64 - 1,
                                    2_812_281 * 768 - 1], dtype=np.uint64)])
    out["rng_keys"] = np.array(keys, dtype=np.uint64)
    out["rng_idx"] = idx
    out["rng_bits"] = np.stack([R.RoundingRng(s).bits(st, t, idx) for s, st, t in keys])
    out["rng_uniform"] = np.stack([R.RoundingRng(s).uniform(st, t, idx) for s, st, t in keys])

    # -- formats.py:197-225: RTN and SR on edge-heavy inputs --------------
    g = np.random.default_rng(11)
    fmts = ["bf16", "e4m3", "e5m2", "fp16", "e3m2", "e2m1"]
    special = np.array([0.0, -0.0, 1.0, -1.0, 17.0, 19.0, 448.0, 449.0, 464.0,
                        465.0, 1e6, -1e6, 2.0**-9, 2.0**-10, 3 * 2.0**-11,
                        -2.0**-12, -1e-30, 1e-30, 1.5 * 2.0**-10, 57344.0,
                        61440.0, 65504.0, 3.3895313892515355e38,
                        -3.3895313892515355e38, 1e-45, -1e-45, 2.0**-133,
                        2.0**-134, 0.1, -0.3], dtype=np.float32)
    rnd = np.concatenate([
        g.normal(scale=1.0, size=400), g.normal(scale=0.02, size=400),
        g.normal(scale=1e-3, size=200), g.normal(scale=300.0, size=200),
        np.ldexp(g.uniform(-1, 1, size=200), g.integers(-140, 120, size=200)),
    ]).astype(np.float32)
    vals = np.concatenate([special, rnd]).astype(np.float32)
    out["fmt_names"] = np.array(fmts)
    out["fmt_inputs"] = vals
    sr_rng = R.RoundingRng(42)
    sr_idx = np.arange(vals.size, dtype=np.uint64) * np.uint64(7919) + np.uint64(3)
    for name in fmts:
        fmt = F.parse_format(name)
        out[f"rtn_{name}"] = F.round_nearest(fmt, vals)
        out[f"sr_{name}"] = F.round_stochastic(fmt, vals, sr_rng, 5, H.HEAD_WEIGHTS_TAG, sr_idx)
        lo, hi = F.neighbors(fmt, vals)
        out[f"lo_{name}"] = lo
        out[f"hi_{name}"] = hi
        out[f"maxfinite_{name}"] = np.float64(fmt.max_finite)
    out["sr_idx"] = sr_idx
    # SR unbiasedness draw: one value, many keys (acceptance-03 style)
    x0 = np.float32(0.3)
    many = np.arange(4096, dtype=np.uint64)
    out["sr_many_e4m3"] = F.round_stochastic(F.E4M3, np.full(4096, x0), sr_rng, 9, 77, many)

    # -- formats.py:246-263: Kahan KAT (test_formats.py:216-229 style) -----
    st = F.KahanState.zeros(4)
    st.sum[:] = F.round_nearest(F.BF16, np.array([1.0, 256.0, -3.0, 0.5], np.float32))
    for _ in range(4096):
        st = F.kahan_add(st, np.full(4, 2.0**-12, np.float32), F.BF16)
    out["kahan_sum"] = st.sum
    out["kahan_comp"] = st.comp

    # -- optimizers.py:51-74: SGD + RTN / SR -------------------------------
    for name in ["bf16", "e4m3"]:
        fmt = F.parse_format(name)
        w = F.round_nearest(fmt, g.normal(scale=0.05, size=(37, 50)).astype(np.float32))
        grad = g.normal(scale=0.3, size=(37, 50)).astype(np.float32)
        gi = (np.arange(37, dtype=np.uint64)[:, None] * np.uint64(768)
              + np.arange(50, dtype=np.uint64)[None, :] + np.uint64(12345))
        out[f"sgd_{name}_w"] = w
        out[f"sgd_{name}_grad"] = grad
        out[f"sgd_{name}_idx"] = gi
        for rmode in ["nearest", "stochastic"]:
            cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding=rmode)
            res = O.sgd_sr_step(F.QuantizedMatrix(w.copy(), fmt), grad, cfg,
                                R.RoundingRng(3), 4, H.HEAD_WEIGHTS_TAG, gi)
            out[f"sgd_{name}_{rmode}"] = res.values

    # -- head.py:51-66 partition / canonical pieces -------------------------
    parts = []
    for total, k in [(64, 8), (100, 7), (5, 8), (1000, 3), (2_812_281, 8), (131_073, 1)]:
        for a, b in H.partition(total, k):
            parts.append((total, k, a, b))
    out["partition"] = np.array(parts, dtype=np.int64)
    pieces = []
    for total, k in [(1000, 3), (300, 2), (4096, 1)]:
        for a, b in H.partition(total, k):
            for s, e in H.canonical_pieces(a, b, total):
                pieces.append((total, k, a, b, s, e))
    out["pieces"] = np.array(pieces, dtype=np.int64)

    # -- head.py:254-298: full head steps at small shapes ------------------
    cases = [("bf16", "nearest", 1, 0.0, 0.0), ("bf16", "stochastic", 3, 1e-4, 0.0),
             ("e4m3", "nearest", 2, 1e-4, 0.0), ("e4m3", "stochastic", 1, 0.0, 0.0),
             ("e4m3", "stochastic", 4, 1e-4, 0.0), ("bf16", "stochastic", 1, 0.0, 0.1),
             ("e4m3", "stochastic", 2, 1e-4, 0.2), ("bf16", "nearest", 3, 1e-4, 0.35)]
    L, d, b = 300, 128, 16
    for ci, (name, rmode, k, wd, p) in enumerate(cases):
        fmt = F.parse_format(name)
        head = H.ChunkedHead.create(L, d, fmt, seed=ci, num_chunks=k, dropout_p=p)
        rs = np.random.default_rng(100 + ci)
        X = rs.normal(size=(b, d)).astype(np.float32)
        labels = [sorted(rs.choice(L, size=rs.integers(1, 5), replace=False).tolist())
                  for _ in range(b)]
        batch = H.BatchInput.from_label_lists(X, labels)
        cfg = O.SgdSrConfig(lr=0.05, weight_decay=wd, fmt=fmt, rounding=rmode)
        rng = R.RoundingRng(ci + 1)
        W0 = head.weights.values.copy()
        # logits / G of the first chunk at step 0, before any update
        Xq = F.round_nearest(fmt, X)
        c0 = head.chunks()[0]
        logits0 = H.head_forward_logits(head, c0, Xq, rng, 0)
        inc = (batch.label_idx >= c0[0]) & (batch.label_idx < c0[1])
        G0 = H.logit_gradient(logits0, batch.sample_idx[inc], batch.label_idx[inc], c0)
        gx1 = H.head_update(head, batch, cfg, rng, 0)
        W1 = head.weights.values.copy()
        gx2 = H.head_update(head, batch, cfg, rng, 1)
        W2 = head.weights.values.copy()
        pre = f"head{ci}_"
        out[pre + "meta"] = np.array([L, d, b, k], dtype=np.int64)
        out[pre + "cfg"] = np.array([0.05, wd, p, ci + 1], dtype=np.float64)
        out[pre + "fmt"] = np.array(name)
        out[pre + "rounding"] = np.array(rmode)
        out[pre + "W0"] = W0
        out[pre + "X"] = X
        out[pre + "sample_idx"] = batch.sample_idx
        out[pre + "label_idx"] = batch.label_idx
        out[pre + "logits0"] = logits0
        out[pre + "G0"] = G0
        out[pre + "gradX1"] = gx1
        out[pre + "W1"] = W1
        out[pre + "gradX2"] = gx2
        out[pre + "W2"] = W2
        out[pre + "ckpt"] = np.frombuffer(_ckpt(H, head), dtype=np.uint8)
    out["head_ncases"] = np.int64(len(cases))

    # -- metrics.py:38-79: top-k with ties ---------------------------------
    sc = np.round(g.normal(size=(6, 40)), 1).astype(np.float32)
    out["topk_scores"] = sc
    out["topk_5"] = np.stack([M.top_k_indices(s, 5) for s in sc])
    truths = [[0, 3, 5], [1], [39, 2], [7, 8, 9, 10], [20], [11, 12]]
    out["topk_truth_flat"] = np.array([t for tt in truths for t in tt])
    out["topk_truth_len"] = np.array([len(t) for t in truths])
    out["p_at_k"] = np.array([M.dataset_precision_at_k(sc, truths, k) for k in (1, 3, 5)])

    path = os.path.join(HERE, "lpxmc_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, lpxmc {lpxmc.__version__})")


def _ckpt(H, head):
    import io
    buf = io.BytesIO()
    H.save_head(head, buf)
    return buf.getvalue()


if __name__ == "__main__":
    main()
