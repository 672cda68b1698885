"""ctypes binding of the C ABI in include/xmc_head.h (libxmc_b200.so).

The product path has no fallback: if the CUDA library is missing or no CUDA
device is present, every entry point raises.  Error codes map onto the
exceptions the reference raises (formats.py / head.py / optimizers.py).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# XMC_LIB_PATH selects another in-tree build (A/B measurements in tools/ab.sh)
LIB_PATH = os.environ.get("XMC_LIB_PATH") or os.path.join(_HERE, "libxmc_b200.so")

XMC_OK = 0
XMC_ERR_ARG = 1
XMC_ERR_SHAPE = 2
XMC_ERR_NONFINITE = 3
XMC_ERR_INDEX = 4
XMC_ERR_LABEL = 5
XMC_ERR_CUDA = 6
XMC_ERR_UNSUPPORTED = 7
XMC_ERR_CAPACITY = 8

FMT_FP32, FMT_BF16, FMT_FP16, FMT_E4M3, FMT_E5M2 = 0, 1, 2, 3, 4
ROUND_NEAREST, ROUND_SR_EXACT, ROUND_SR_FAST = 0, 1, 2
PRECISION_OPERAND, PRECISION_REFERENCE = 0, 1


class HeadDesc(ctypes.Structure):
    _fields_ = [("num_labels_global", ctypes.c_int64), ("label_offset", ctypes.c_int64),
                ("num_labels_local", ctypes.c_int64), ("dim", ctypes.c_int32),
                ("fmt", ctypes.c_int32), ("num_chunks", ctypes.c_int32),
                ("max_batch", ctypes.c_int32), ("max_positives", ctypes.c_int64),
                ("num_sms", ctypes.c_int32), ("comp_bytes", ctypes.c_int32),
                ("dropout", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("comp_labels", ctypes.c_int64), ("g_format", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class StepArgs(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("rounding", ctypes.c_int32), ("sr_bits", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("step", ctypes.c_uint64),
                ("tensor_id", ctypes.c_uint64), ("dropout_p", ctypes.c_double)]


class AdamWArgs(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("weight_decay", ctypes.c_float), ("eps", ctypes.c_float),
                ("reserved", ctypes.c_float), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("t", ctypes.c_int64)]


class Grid(ctypes.Structure):
    _fields_ = [("exp_bits", ctypes.c_int32), ("man_bits", ctypes.c_int32),
                ("extended_range", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32, _I64, _U64, _F32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float

_SIGNATURES = {
    "xmc_last_error": ([], ctypes.c_char_p),
    "xmc_version": ([], ctypes.c_char_p),
    "xmc_head_workspace_size": ([ctypes.POINTER(HeadDesc), ctypes.POINTER(ctypes.c_size_t)], _I32),
    "xmc_head_create": ([ctypes.POINTER(HeadDesc), _P, ctypes.c_size_t, ctypes.POINTER(_P)], _I32),
    "xmc_head_destroy": ([_P], _I32),
    "xmc_peer_create": ([_I32, _I32, _I32, _I32, ctypes.POINTER(_P), _P], _I32),
    "xmc_peer_connect": ([_P, _P], _I32),
    "xmc_peer_destroy": ([_P], _I32),
    "xmc_head_attach_peers": ([_P, _P], _I32),
    "xmc_head_step": ([_P, _P, _P, _I32, _P, _P, _I64, ctypes.POINTER(StepArgs), _P, _P, _P], _I32),
    "xmc_head_step_kahan": ([_P, _P, _P, _P, _I32, _P, _P, _I64, ctypes.POINTER(StepArgs), _P, _P, _P], _I32),
    "xmc_head_check": ([_P, _P], _I32),
    "xmc_head_logits": ([_P, _P, _P, _I32, _I64, _I64, _P, _I64, ctypes.POINTER(StepArgs), _P], _I32),
    "xmc_head_topk": ([_P, _P, _P, _I32, _I32, _P, _P, _P], _I32),
    "xmc_dropout_mask": ([_I64, _I64, _I32, _U64, _U64, ctypes.c_double, _P, _P], _I32),
    "xmc_logit_gradient": ([_P, _I64, _I32, _I64, _P, _P, _I64, _I64, _P, _P], _I32),
    "xmc_head_backward": ([_P, _P, _P, _I64, _P, _I32, _I64, _I64, _P, _I32, _I32,
                           ctypes.POINTER(StepArgs), _P], _I32),
    "xmc_round_nearest": ([Grid, _P, _P, _I64, _P], _I32),
    "xmc_round_stochastic": ([Grid, _P, _P, _I64, _U64, _U64, _U64, _P, _P], _I32),
    "xmc_sgd_sr_step": ([Grid, _P, _P, _I64, _F32, _F32, _I32, _U64, _U64, _U64, _P, _P, _P], _I32),
    "xmc_kahan_sgd_step": ([Grid, _P, _P, _P, _I64, _F32, _F32, _I32, _U64, _U64, _U64, _P, _P, _P],
                           _I32),
    "xmc_cast_rn": ([_P, _P, _I64, _I32, _P, _P], _I32),
    "xmc_head_step_adamw": ([_P, _P, _P, _P, _P, _P, _I32, _P, _P, _I64, ctypes.POINTER(AdamWArgs),
                             ctypes.POINTER(StepArgs), _P, _P, _P], _I32),
    "xmc_kahan_adamw_step": ([Grid, _P, _P, _P, _P, _P, _I64, _F32, ctypes.c_double, ctypes.c_double, _F32, _F32,
                              _I64, _P], _I32),
    "xmc_profile_enable": ([_I32], _I32),
    "xmc_profile_read": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64),
                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)], _I32),
    "xmc_profile_clock": ([ctypes.POINTER(ctypes.c_uint64)], _I32),
}


def profile_enable(on: bool):
    load().xmc_profile_enable(1 if on else 0)


def profile_read():
    """-> (ms_fwd, n_fwd, ms_bwd, n_bwd) since the previous read."""
    a, b = ctypes.c_double(), ctypes.c_double()
    na, nb = _I64(), _I64()
    load().xmc_profile_read(ctypes.byref(a), ctypes.byref(na), ctypes.byref(b), ctypes.byref(nb))
    return a.value, na.value, b.value, nb.value



def profile_clock():
    """-> {"fwd": MHz or None, "bwd": MHz or None}: effective SM clock of the
    fwd / bwd launches since the previous read (block 0's clock64 / globaltimer)."""
    out = (ctypes.c_uint64 * 4)()
    check(load().xmc_profile_clock(out))
    res = {}
    for k, i in (("fwd", 0), ("bwd", 2)):
        res[k] = out[i] / out[i + 1] * 1e3 if out[i + 1] else None
    return res

_lib = None


def load():
    """Load libxmc_b200.so (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                               "(there is no CPU fallback for the head)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def exported_symbols():
    return list(_SIGNATURES)


def check(status: int):
    if status == XMC_OK:
        return
    msg = load().xmc_last_error().decode("utf-8", "replace")
    if status in (XMC_ERR_ARG, XMC_ERR_SHAPE, XMC_ERR_NONFINITE, XMC_ERR_LABEL):
        raise ValueError(msg)
    if status == XMC_ERR_INDEX:
        raise IndexError(msg)
    if status == XMC_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"xmc error {status}: {msg}")


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
