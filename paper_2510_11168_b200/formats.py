"""Float grids and device rounding -- mirror of lpxmc.formats / lpxmc.rng.

Grid descriptors are pure host metadata (formats.py:49-156); the rounding
functions run on the GPU through the C ABI and are bit-exact with the
reference (round_nearest formats.py:197-206, round_stochastic :209-225,
keyed draws rng.py:36-57).  Values live in float32 tensors on the grid, the
same convention as the reference's QuantizedMatrix (formats.py:306-327);
the head itself stores weights in the native torch dtype instead.
"""

from __future__ import annotations

from dataclasses import dataclass, field
import re

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class FloatFormat:
    """formats.py:49-137."""

    exp_bits: int
    man_bits: int
    saturating: bool = True
    extended_range: bool | None = field(default=None)

    def __post_init__(self):
        if not (2 <= self.exp_bits <= 8):
            raise ValueError(f"exp_bits must be in [2, 8], got {self.exp_bits}")
        if not (0 <= self.man_bits <= 23):
            raise ValueError(f"man_bits must be in [0, 23], got {self.man_bits}")
        if self.extended_range is None:
            object.__setattr__(self, "extended_range", (self.exp_bits, self.man_bits) == (4, 3))

    @property
    def bias(self) -> int:
        return 2 ** (self.exp_bits - 1) - 1

    @property
    def min_normal_exp(self) -> int:
        return 1 - self.bias

    @property
    def max_exp(self) -> int:
        return self.bias + 1 if self.extended_range else self.bias

    @property
    def min_exp(self) -> int:
        return self.min_normal_exp - self.man_bits

    @property
    def max_finite(self) -> float:
        if self.extended_range:
            if self.man_bits == 0:
                raise ValueError("extended range needs at least one mantissa bit")
            top = 2.0 - 2.0 ** (1 - self.man_bits)
        else:
            top = 2.0 - 2.0 ** (-self.man_bits)
        return float(top * 2.0 ** self.max_exp)

    @property
    def storage_bits(self) -> int:
        return 1 + self.exp_bits + self.man_bits

    @property
    def name(self) -> str:
        named = {(8, 23): "fp32", (8, 7): "bf16", (5, 10): "fp16", (4, 3): "e4m3", (5, 2): "e5m2"}
        return named.get((self.exp_bits, self.man_bits), f"e{self.exp_bits}m{self.man_bits}")

    @property
    def is_working_precision(self) -> bool:
        return self.exp_bits == 8 and self.man_bits == 23

    # --- B200 additions -------------------------------------------------
    @property
    def torch_dtype(self):
        """Native storage dtype; bit patterns equal encode_grid_bits (head.py:317-338)."""
        return {"bf16": torch.bfloat16, "e4m3": torch.float8_e4m3fn,
                "e5m2": torch.float8_e5m2, "fp16": torch.float16,
                "fp32": torch.float32}.get(self.name)

    @property
    def code(self) -> int:
        return {"fp32": _lib.FMT_FP32, "bf16": _lib.FMT_BF16, "fp16": _lib.FMT_FP16,
                "e4m3": _lib.FMT_E4M3, "e5m2": _lib.FMT_E5M2}.get(self.name, -1)

    def grid(self) -> _lib.Grid:
        if not self.saturating:
            raise NotImplementedError("non-saturating grids are not supported on the GPU path")
        return _lib.Grid(self.exp_bits, self.man_bits, 1 if self.extended_range else 0, 0)


FP32 = FloatFormat(8, 23)
BF16 = FloatFormat(8, 7)
FP16 = FloatFormat(5, 10)
E4M3 = FloatFormat(4, 3)
E5M2 = FloatFormat(5, 2)
_NAMED = {"fp32": FP32, "bf16": BF16, "fp16": FP16, "e4m3": E4M3, "e5m2": E5M2}


def parse_format(name: str) -> FloatFormat:
    """formats.py:148-156."""
    key = name.strip().lower()
    if key in _NAMED:
        return _NAMED[key]
    m = re.fullmatch(r"e(\d+)m(\d+)", key)
    if m is None:
        raise ValueError(f"unknown float format {name!r}")
    return FloatFormat(int(m.group(1)), int(m.group(2)))


def _f32_cuda(x) -> torch.Tensor:
    t = torch.as_tensor(x, dtype=torch.float32)
    if not t.is_cuda:
        t = t.cuda()
    return t.contiguous()


def _index_tensor(index, n, device):
    """Flat uint64 keys as a device int64 tensor holding the same 8 bytes."""
    if index is None:
        return None
    if isinstance(index, torch.Tensor):
        t = index.reshape(-1)
        t = t.view(torch.int64) if t.dtype == torch.uint64 else t.to(torch.int64)
    else:
        a = np.ascontiguousarray(np.asarray(index, dtype=np.uint64).reshape(-1))
        t = torch.from_numpy(a.view(np.int64))
    if t.numel() == 1 and n != 1:
        t = t.expand(n)
    if t.numel() != n:
        raise ValueError("index shape does not match x")
    return t.to(device).contiguous()


def round_nearest(fmt: FloatFormat, x) -> torch.Tensor:
    """RTN ties-to-even onto fmt's grid (formats.py:197-206), on the GPU."""
    t = _f32_cuda(x)
    out = torch.empty_like(t)
    _lib.check(_lib.load().xmc_round_nearest(fmt.grid(), t.data_ptr(), out.data_ptr(), t.numel(),
                                             _lib.stream_ptr()))
    return out


def round_stochastic(fmt: FloatFormat, x, rng, step: int, tensor_id: int, index=None) -> torch.Tensor:
    """SR with the reference's keyed splitmix64 draws (formats.py:209-225)."""
    t = _f32_cuda(x)
    out = torch.empty_like(t)
    idx = _index_tensor(index, t.numel(), t.device)
    _lib.check(_lib.load().xmc_round_stochastic(
        fmt.grid(), t.data_ptr(), out.data_ptr(), t.numel(), rng.seed, step & (2**64 - 1),
        tensor_id & (2**64 - 1), _lib.ptr(idx), _lib.stream_ptr()))
    return out


# ----------------------------------------------------------------- rng.py

def tensor_tag(name: str) -> int:
    """FNV-1a 64 (rng.py:28-33)."""
    h = 0xCBF29CE484222325
    for b in name.encode("utf-8"):
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


class RoundingRng:
    """Key holder for the device generator (rng.py:36-57).  Draws are made
    inside the kernels from (seed, step, tensor_id, flat index)."""

    def __init__(self, seed: int):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
