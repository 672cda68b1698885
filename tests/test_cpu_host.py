"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares (no compute without a GPU), and the host-side mirror of the
reference interface agrees with the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import lpxmc_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    from paper_2510_11168_b200 import _build, _lib
    _build.build()
    lib = _lib.load()
    hdr = open(os.path.join(ROOT, "include", "xmc_head.h")).read()
    names = set(re.findall(r"\b(xmc_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 16
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert set(_lib.exported_symbols()) == names
    assert lib.xmc_version().startswith(b"xmc-b200")


def test_host_errors_without_device_work():
    """Argument validation happens before any CUDA call."""
    import ctypes
    from paper_2510_11168_b200 import _lib
    lib = _lib.load()
    size = ctypes.c_size_t()
    bad = _lib.HeadDesc(100, 0, 100, 100, _lib.FMT_E4M3, 1, 16, 10, 148, 0)   # dim % 128 != 0
    assert lib.xmc_head_workspace_size(ctypes.byref(bad), ctypes.byref(size)) == _lib.XMC_ERR_SHAPE
    bad = _lib.HeadDesc(100, 50, 100, 128, _lib.FMT_E4M3, 1, 16, 10, 148, 0)  # shard past L
    assert lib.xmc_head_workspace_size(ctypes.byref(bad), ctypes.byref(size)) == _lib.XMC_ERR_ARG
    bad = _lib.HeadDesc(100, 0, 100, 128, _lib.FMT_FP16, 1, 16, 10, 148, 0)   # unsupported storage
    assert lib.xmc_head_workspace_size(ctypes.byref(bad), ctypes.byref(size)) == _lib.XMC_ERR_UNSUPPORTED
    ok = _lib.HeadDesc(2_812_281, 0, 2_812_281, 768, _lib.FMT_E4M3, 8, 256, 20000, 148, 0)
    assert lib.xmc_head_workspace_size(ctypes.byref(ok), ctypes.byref(size)) == _lib.XMC_OK
    # C4 workspace: G chunk (351,536 x 256 e4m3) + grad_X partials + lists: well under 200 MB
    assert 90e6 < size.value < 200e6
    with pytest.raises(ValueError):
        _lib.check(_lib.XMC_ERR_NONFINITE)
    with pytest.raises(IndexError):
        _lib.check(_lib.XMC_ERR_INDEX)


def test_host_mirror_matches_oracle():
    import paper_2510_11168_b200 as xmc
    for total, k in [(64, 8), (100, 7), (5, 8), (2_812_281, 8)]:
        assert xmc.partition(total, k) == O.partition(total, k)
    for a, b, total in [(0, 333, 1000), (333, 666, 1000), (10, 20, 100)]:
        assert xmc.canonical_pieces(a, b, total) == O.canonical_pieces(a, b, total)
    assert xmc.HEAD_WEIGHTS_TAG == O.HEAD_WEIGHTS_TAG and xmc.DROPOUT_TAG == O.DROPOUT_TAG
    for name in ["bf16", "e4m3", "e5m2", "fp16", "fp32", "e3m2"]:
        a, b = xmc.parse_format(name), O.parse_format(name)
        assert (a.max_finite, a.min_exp, a.max_exp, a.name) == (b.max_finite, b.min_exp, b.max_exp, b.name)
    with pytest.raises(ValueError):
        xmc.SgdSrConfig(lr=0.0)
    with pytest.raises(ValueError):
        xmc.SgdSrConfig(lr=0.1, rounding="up")
    with pytest.raises(ValueError):
        xmc.parse_format("q7")


def test_positive_bucketing_host_model():
    """The device buckets positives by (chunk, 128-label tile); restate the
    geometry on the host and check it covers every in-shard label once."""
    L, k = 10_007, 3
    chunks = O.partition(L, k)
    tile_base, tb = [], 0
    for s, e in chunks:
        tile_base.append(tb)
        tb += -(-(e - s) // 128)
    labels = np.arange(L)
    seen = np.zeros(tb * 128, bool)
    for lab in labels:
        c = min(lab * k // L, k - 1)
        while c > 0 and chunks[c][0] > lab:
            c -= 1
        while c + 1 < k and chunks[c + 1][0] <= lab:
            c += 1
        off = lab - chunks[c][0]
        slot = (tile_base[c] + off // 128) * 128 + off % 128
        assert not seen[slot]
        seen[slot] = True
    assert seen.sum() == L


def test_peer_group_argument_checks_without_device():
    """xmc_peer_create validates rank / world / dim / batch before any CUDA
    call, and the step-args generator field is range-checked (no GPU here)."""
    import ctypes
    from paper_2510_11168_b200 import _lib
    from paper_2510_11168_b200.optimizers import SgdSrConfig
    lib = _lib.load()
    p = ctypes.c_void_p()
    h = (ctypes.c_char * 64)()
    hv = ctypes.cast(h, ctypes.c_void_p)
    assert lib.xmc_peer_create(0, 0, 768, 256, ctypes.byref(p), hv) == _lib.XMC_ERR_ARG      # world 0
    assert lib.xmc_peer_create(2, 2, 768, 256, ctypes.byref(p), hv) == _lib.XMC_ERR_ARG      # rank >= world
    assert lib.xmc_peer_create(0, 9, 768, 256, ctypes.byref(p), hv) == _lib.XMC_ERR_ARG      # > 8 ranks
    assert lib.xmc_peer_create(0, 2, 100, 256, ctypes.byref(p), hv) == _lib.XMC_ERR_SHAPE    # dim % 128
    assert lib.xmc_peer_create(0, 2, 768, 65536, ctypes.byref(p), hv) == _lib.XMC_ERR_ARG    # batch > 65535
    assert lib.xmc_peer_connect(None, hv) == _lib.XMC_ERR_ARG
    assert lib.xmc_head_attach_peers(None, None) == _lib.XMC_ERR_ARG
    # SgdSrConfig: generator names map onto (rounding code, sr_bits)
    from paper_2510_11168_b200.formats import E4M3
    assert (SgdSrConfig(0.1, fmt=E4M3).rounding_code, SgdSrConfig(0.1, fmt=E4M3).sr_bits) == (_lib.ROUND_SR_FAST, 0)
    c = SgdSrConfig(0.1, fmt=E4M3, sr_impl="philox")
    assert (c.rounding_code, c.sr_bits) == (_lib.ROUND_SR_FAST, 1)
    c = SgdSrConfig(0.1, fmt=E4M3, sr_impl="splitmix64")
    assert c.rounding_code == _lib.ROUND_SR_EXACT
    with pytest.raises(ValueError):
        SgdSrConfig(0.1, fmt=E4M3, sr_impl="xorshift")


def test_integration_stub_matches_the_abi():
    """INTEGRATION.md's reference-side ctypes stub declares xmc_head_desc /
    xmc_step_args with the same fields, in the same order, as the binding the
    package uses (paper_2510_11168_b200/_lib.py)."""
    import re
    from paper_2510_11168_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()

    def fields(cls_name):
        m = re.search(r"class " + cls_name + r"\(ctypes\.Structure\):\s*_fields_ = \[(.*?)\]\n", text, re.S)
        assert m, cls_name
        return [(n, getattr(ctypes, t)) for n, t in re.findall(r'\("(\w+)", ctypes\.(\w+)\)', m.group(1))]

    assert fields("_Desc") == list(_lib.HeadDesc._fields_)
    assert fields("_Step") == list(_lib.StepArgs._fields_)


def test_bench_reference_arm_line():
    """`bench.py --impl reference` (the driver's reference arm) runs on the
    host cores without a GPU and prints the contract's JSON line."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-seconds", "0.5", "--cpu-labels", "512"],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    d = json.loads(out.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["labels"] == 2_812_281 and d["metric"] == "head train samples/sec at 3M labels FP8"
