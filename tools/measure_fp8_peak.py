"""Measure the dense FP8 (e4m3) tensor-core peak of this B200 with cuBLASLt
(torch._scaled_mm), the FP8 counterpart of MEASURED_PEAKS.json's bf16 number.
Writes profiles/fp8_peak.json: burst (best of 10) and sustained (back to back
for ~4 s) TFLOP/s of an 8192^3 GEMM, plus the clocks seen."""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    n = 8192
    dev = torch.device("cuda", 0)
    a = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn)
    b = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn).t()  # column-major operand
    one = torch.tensor(1.0, device=dev)
    mm = lambda: torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
    for _ in range(5):
        mm()
    torch.cuda.synchronize()
    flops = 2.0 * n ** 3
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mm()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = max(10, int(4000 / best))
    e0.record()
    for _ in range(iters):
        mm()
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / iters
    out = {"tflops": flops / (best * 1e-3) / 1e12, "tflops_sustained": flops / (sus * 1e-3) / 1e12,
           "how": "torch._scaled_mm e4m3 x e4m3 -> bf16, 8192^3 (2 N^3 flops); burst = best of 10, "
                  f"sustained = {iters} back-to-back launches",
           "gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    path = os.path.join(ROOT, "profiles", "fp8_peak.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
