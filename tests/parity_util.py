"""Shared checkers of the GPU parity tests (test infrastructure)."""

import numpy as np
import torch

from oracle import lpxmc_oracle as O


def ulp_dist(a, b, fmt):
    """|a - b| in units of fmt's grid spacing at the larger magnitude."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / O._ulp_of(fmt, np.maximum(np.abs(a), np.abs(b)))


def fp32_update_noise(lr, G, Xq):
    """lr * gamma * ((|G| + Y) @ |Xq|): the fp32 evaluation-order bound of an
    update value (see reference_weight_report)."""
    Ga = np.abs(np.asarray(G, np.float64)) + (np.asarray(G) < 0)
    gamma = (4 * np.asarray(Xq).shape[0] + 16) * 2.0 ** -24
    return lr * gamma * (Ga @ np.abs(np.asarray(Xq, np.float64)))


def reference_weight_report(got, ref, fmt, lr, G, Xq, sr=False):
    """Weights of the reference-precision mode against the UNMODIFIED
    reference / oracle (fp32 G in both GEMMs).  The two sides multiply the
    same exact products and differ only in fp32 evaluation order (tensor-core
    vs OpenBLAS accumulation, CUDA vs numpy expf in G: a few fp32 ulps of the
    update value), so an element may differ only where that noise straddles a
    grid rounding boundary.  Returns (fraction bit-identical, fraction more
    than one grid ulp apart, and whether every element lies within
        one grid ulp + lr * gamma * ((|G| + Y) @ |Xq|),
    gamma = (4 B + 16) 2^-24: the worst-case fp32 summation error of the two
    dot products (Higham's gamma_n = n u; the GPU sums 3 B exact products of
    the bf16 planes, the reference B, plus the few ulps of G itself).  It
    only matters where the update cancels W to far below its own terms.  Y (1
    at positives) covers the positives' sigmoid - 1, whose absolute error is
    that of sigmoid ~ 1.  With stochastic rounding (sr=True) the noise can
    also move the update across a grid point, which changes its neighbour
    pair: two grid ulps."""
    got = np.asarray(got, np.float32)
    ref = np.asarray(ref, np.float32)
    same = float(np.mean(got.view(np.uint32) == ref.view(np.uint32)))
    du = ulp_dist(got, ref, fmt)
    noise = fp32_update_noise(lr, G, Xq)
    ulp = O._ulp_of(fmt, np.maximum(np.abs(got), np.abs(ref)).astype(np.float64))
    bound = (2.0 if sr else 1.0) * ulp + noise + 1e-30
    ratio = np.abs(got.astype(np.float64) - ref) / bound
    ok = bool(np.all(ratio <= 1.0))
    if not ok:
        i = np.unravel_index(int(np.argmax(ratio)), ratio.shape)
        print(f"worst element {i}: got {got[i]!r} ref {ref[i]!r} ulp {ulp[i]:.3e} noise {noise[i]:.3e} "
              f"ratio {ratio[i]:.2f}; {int((ratio > 1).sum())} elements over the bound")
    return same, float(np.mean(du > 1.0 + 1e-9)), ok


def torch_fp32_grad_x(W, Xq, si, li, label0=0, slab=131_072, logit_scale=1.0):
    """fp32 restatement of head_update's grad_X (head.py:181-209) on the GPU
    for full-size checks: G = clip(sigmoid(W Xq^T)) - Y per label slab,
    acc += G^T W, TF32 off.  W: (L, d) native tensor on the device, Xq: (B, d)
    on-grid fp32 numpy, positives as GLOBAL labels (label0 = W's first row)."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        dev = W.device
        Xt = torch.from_numpy(np.ascontiguousarray(Xq)).to(dev)
        B = Xt.shape[0]
        acc = torch.zeros((B, W.shape[1]), dtype=torch.float64, device=dev)
        si_t = torch.from_numpy(np.asarray(si, np.int64)).to(dev)
        li_t = torch.from_numpy(np.asarray(li, np.int64)).to(dev) - label0
        for r0 in range(0, W.shape[0], slab):
            r1 = min(W.shape[0], r0 + slab)
            w = W[r0:r1].float()
            z = (w @ Xt.T) * logit_scale
            g = torch.clamp(torch.sigmoid(z), 2.0 ** -24, 1.0 - 2.0 ** -24)
            m = (li_t >= r0) & (li_t < r1)
            g[li_t[m] - r0, si_t[m]] -= 1.0
            acc += (g.T @ w).double()
        return acc.float()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
