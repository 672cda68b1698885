"""Benchmark of the ELMO head step on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[3]): Amazon-3M shape,
L = 2,812,281 labels, d = 768, batch 256, FP8 e4m3 weights, SR on (keyed hash
words + cvt.rs), lr 0.05, wd 1e-4, dropout 0, synthetic data: W0 ~ N(0, 0.02^2)
RTN to e4m3, X ~ N(0, 1), positives per sample max(1, Poisson(36.17)) distinct
labels drawn Zipf(1.0).  Labels are sharded contiguously across ranks (strong
scaling: the 3M-label problem is fixed, each rank owns L/N rows).

The headline runs the production operand precision (all three GEMMs on FP8
tensor cores, G as e5m2(2^8 g)); `reference_precision` in the same line is the
same step with the reference's fp32 G (ChunkedHead(precision="reference")).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0).  `value` is device-timed samples/s with inputs
resident in HBM (W = 2.16 GB >> L2, so no flush is needed); `e2e` is the same
metric through the public API with host inputs copied in and grad_X copied
out every step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_MEAN_LABELS = {2_812_281: 36.17, 670_091: 5.45, 131_073: 5.15, 8_623_847: 9.03}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--labels", type=int, default=2_812_281)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--fmt", default="e4m3")
    # label chunks per rank (the reference's memory knob, head.num_chunks).
    # Default: the fewest chunks of at most --max-chunk-rows rows each, so the
    # G buffer per GPU stays the same at every N (C4: k=2 on 1 GPU, k=1 per
    # rank on 2-8 GPUs; fewer, larger chunks have fewer launch tails)
    ap.add_argument("--chunks", type=int, default=None)
    ap.add_argument("--max-chunk-rows", type=int, default=1_406_141)
    ap.add_argument("--rounding", default="stochastic")
    ap.add_argument("--sr-impl", default="hash", choices=["hash", "philox", "splitmix64"])
    ap.add_argument("--precision", default="operand", choices=["operand", "reference"])
    ap.add_argument("--g-format", default="e5m2", choices=["e5m2", "e4m3", "bf16"])
    ap.add_argument("--kahan", default=None, choices=["bf16", "fp32"],
                    help="head-Kahan compensation (PAPER.md:795), fused into the backward")
    ap.add_argument("--kahan-labels", type=int, default=None,
                    help="top-p%% head-Kahan: only the first N (frequency-sorted) labels carry a compensation")
    ap.add_argument("--ref-steps", type=int, default=5,
                    help="timed steps of the reference-precision mode reported beside the headline (0: skip)")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--bf16g-steps", type=int, default=5,
                    help="timed steps of the bf16-G mode (the paper's BF16 logit gradients) reported beside "
                         "the headline (0: skip)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-labels", type=int, default=8192)
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------- synthetic data

def synthetic_positives(num_labels, batch, mean_labels, seed=0):
    """max(1, Poisson(mean)) distinct labels per sample, Zipf(1.0) over [0, L)."""
    rng = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, num_labels + 1, dtype=np.float64)
    cdf = np.cumsum(p)
    cdf /= cdf[-1]
    rows, cols = [], []
    for i in range(batch):
        n = min(max(1, int(rng.poisson(mean_labels))), num_labels)
        chosen = set()
        while len(chosen) < n:
            for lab in np.minimum(np.searchsorted(cdf, rng.random(2 * n), side="right"), num_labels - 1):
                if len(chosen) < n:
                    chosen.add(int(lab))
        for lab in sorted(chosen):
            rows.append(i)
            cols.append(lab)
    return np.array(rows, np.int64), np.array(cols, np.int64)


# ------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled DURING the timed
    region by a separate process polling NVML every ~1 ms (a thread of this
    process would share the GIL with the launch loop and get a sample or two
    in a tens-of-ms region); nvidia-smi -lms 100 as the fallback."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    POLL = r"""
import sys, time, pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
out = []
import select
while True:
    r, _, _ = select.select([sys.stdin], [], [], 0.001)
    if r:
        break
    try:
        out.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                    nv.nvmlDeviceGetCurrentClocksEventReasons(h),
                    nv.nvmlDeviceGetPowerUsage(h) / 1000.0))
    except Exception:
        pass
for s in out:
    print(*s)
"""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []

    def start(self):
        try:
            import pynvml  # noqa: F401  (the poller needs it)
            self.proc = subprocess.Popen([sys.executable, "-c", self.POLL, str(self.index)], stdin=subprocess.PIPE,
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline().split()
            if len(first) == 2 and first[0] == "max":
                self.nvml = True
                self.smax = int(first[1])
                return
            self.proc.kill()
        except Exception:
            pass
        self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            out, _ = self.proc.communicate(input="stop\n", timeout=30)
            samples = []
            for ln in out.splitlines():
                f = ln.split()
                if len(f) == 3:
                    samples.append((int(f[0]), int(f[1]), float(f[2])))
            sm = [s[0] for s in samples]
            reasons = sorted({n for _, rs, _ in samples for n, bit in self.REASONS.items() if rs & bit})
            pw = [s[2] for s in samples]
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_min_mhz": min(sm) if sm else None,
                    "sm_max_mhz": self.smax, "reasons": reasons, "samples": len(sm),
                    "power_w_median": statistics.median(pw) if pw else None,
                    "power_w_max": max(pw) if pw else None, "source": "nvml ~1 ms poll (separate process)"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


# ------------------------------------------------------------- peaks

def fp8_gemm_peak():
    path = os.path.join(ROOT, "profiles", "fp8_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("tflops")
    return None


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    if os.path.exists(path):
        with open(path) as f:
            peaks.update(json.load(f))
        peaks["source"] = "measured"
    fp8 = os.path.join(ROOT, "profiles", "fp8_peak.json")
    if os.path.exists(fp8):
        with open(fp8) as f:
            peaks["fp8"] = json.load(f)
    return peaks


# ------------------------------------------------------------- CPU baseline

def cpu_baseline(a, seconds):
    """The reference algorithm (oracle/lpxmc_oracle.py, numpy restatement of
    lpxmc.head.head_update) on a bounded label slice of the same workload,
    extrapolated linearly in L (time is linear in L)."""
    from oracle import lpxmc_oracle as O
    Ls = min(a.cpu_labels, a.labels)
    fmt = O.parse_format(a.fmt)
    rs = np.random.default_rng(0)
    W = O.round_nearest(fmt, rs.normal(scale=0.02, size=(Ls, a.dim)).astype(np.float32))
    X = rs.normal(size=(a.batch, a.dim)).astype(np.float32)
    mean = PAPER_MEAN_LABELS.get(a.labels, 5.0)
    si, li = synthetic_positives(a.labels, a.batch, mean, seed=1)
    keep = li < Ls
    head = O.OracleHead(W, fmt, max(1, round(a.chunks * Ls / a.labels)))
    cfg = O.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding=a.rounding)
    rng = O.RoundingRng(0)
    O.head_update(head, X, si[keep], li[keep], cfg, rng, 0)  # warm-up
    times, step = [], 1
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 2:
        t0 = time.perf_counter()
        O.head_update(head, X, si[keep], li[keep], cfg, rng, step)
        times.append(time.perf_counter() - t0)
        step += 1
    t_slice = statistics.median(times)
    t_full = t_slice * a.labels / Ls
    return {"value": a.batch / t_full, "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle head_update on {Ls} of {a.labels} labels (d={a.dim}, B={a.batch}, {a.fmt}, "
                      f"{a.rounding}), median of {len(times)} steps = {t_slice:.3f} s, x{a.labels / Ls:.1f} "
                      f"linear in L; numpy/OpenBLAS on {os.cpu_count()} host threads",
            "s_per_step_full": t_full}


# ------------------------------------------------------------- main

def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "head train samples/sec at 3M labels FP8"
    if a.chunks is None:
        shard_rows = -(-a.labels // world)
        a.chunks = max(1, -(-shard_rows // a.max_chunk_rows))
    config = {"workload": f"Amazon-3M head step: L={a.labels}, d={a.dim}, B={a.batch}, {a.fmt} weights, "
                          f"k={a.chunks} chunks, SR={a.rounding}/{a.sr_impl}, lr=0.05, wd=1e-4",
              "labels": a.labels, "dim": a.dim, "global_batch": a.batch, "chunks": a.chunks,
              "precision": a.precision, "g_format": a.g_format if a.fmt == "e4m3" else "bf16",
              "parallelism": f"label-shard x{world}", "l2": "inputs larger than L2 (W >> 126 MB)",
              "cpu_sample_labels": min(a.cpu_labels, a.labels)}
    if a.kahan:
        config["kahan"] = {"comp": a.kahan, "labels": a.kahan_labels or a.labels}

    if a.impl == "reference":
        if rank != 0:
            return
        cb = cpu_baseline(a, a.cpu_seconds)
        out = {"impl": "reference", "metric": metric, "value": cb["value"], "unit": "samples/s",
               "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": a.fmt, "data": "synthetic",
               "config": config, "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
               "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    import torch
    import torch.distributed as dist
    import paper_2510_11168_b200 as xmc
    from paper_2510_11168_b200 import _lib

    # test hook (XMC_BENCH_ONE_DEVICE=1): every rank on cuda:0 with gloo, so the
    # multi-rank flow (peer all-reduce, fallbacks, max-over-ranks timing) runs
    # on a one-GPU box; its timings are meaningless (the ranks time-slice)
    one_dev = os.environ.get("XMC_BENCH_ONE_DEVICE") == "1"
    local = 0 if one_dev else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    lo, hi = xmc.partition(a.labels, world)[rank]
    fmt = xmc.parse_format(a.fmt)

    # weights: N(0, 0.02^2) generated on device in blocks and RTN-cast to the grid
    W = torch.empty((hi - lo, a.dim), dtype=fmt.torch_dtype, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    blk = 262_144
    for r0 in range(0, hi - lo, blk):
        r1 = min(r0 + blk, hi - lo)
        W[r0:r1] = xmc.cast_native(torch.randn((r1 - r0, a.dim), generator=g, device=dev) * 0.02, fmt)
    head = xmc.ChunkedHead(xmc.QuantizedMatrix(W, fmt), num_chunks=a.chunks, num_labels_global=a.labels,
                           label_offset=lo, precision=a.precision, g_format=a.g_format,
                           kahan=a.kahan, kahan_labels=a.kahan_labels)
    rs = np.random.default_rng(0)
    Xh = rs.normal(size=(a.batch, a.dim)).astype(np.float32)
    si, li = synthetic_positives(a.labels, a.batch, PAPER_MEAN_LABELS.get(a.labels, 5.0), seed=1)
    cfg = xmc.SgdSrConfig(lr=0.05, weight_decay=1e-4, fmt=fmt, rounding=a.rounding, sr_impl=a.sr_impl)
    rng = xmc.RoundingRng(0)
    Xd = torch.from_numpy(Xh).to(dev)
    sid = torch.from_numpy(si.astype(np.int32)).to(dev)
    lid = torch.from_numpy(li.astype(np.int32)).to(dev)
    batch_dev = xmc.BatchInput(Xd, sid, lid)
    gx = torch.empty((a.batch, a.dim), dtype=torch.float32, device=dev)

    # grad_X across ranks: the peer-memory all-reduce fused into the step's own
    # grad_X reduction (parallel.PeerGroup; XMC_PEER=0 -> NCCL all_reduce)
    allreduce = "none (1 rank)"
    peers = None
    if world > 1:
        allreduce = "gloo all_reduce (one-device test hook)" if one_dev else "nccl all_reduce"
        if os.environ.get("XMC_PEER", "1") != "0":
            from paper_2510_11168_b200.parallel import PeerGroup
            try:
                peers = PeerGroup(a.dim, a.batch)
                peers.attach(head)
                allreduce = "peer memory (CUDA IPC over NVLink), fused with the partial-slot reduction"
            except Exception as e:  # noqa: BLE001 - report and keep NCCL
                print(f"peer all-reduce unavailable ({e}); using NCCL", file=sys.stderr)
                peers = None
    gx_allreduce = [allreduce]

    def step_fn(s, batch, out):
        r = xmc.head_update(head, batch, cfg, rng, s, check=False, grad_out=out)
        if world > 1 and head.peers is None:
            dist.all_reduce(r)
        return r

    torch.cuda.reset_peak_memory_stats(dev)
    mem0 = torch.cuda.memory_allocated(dev)
    for s in range(a.warmup):
        step_fn(s, batch_dev, gx)
    ok = True
    try:
        _lib.check(_lib.load().xmc_head_check(head.handle(a.batch, len(si)).h, _lib.stream_ptr()))
    except Exception as e:  # noqa: BLE001
        if peers is None:
            raise
        print(f"peer all-reduce failed in warm-up ({e}); using NCCL", file=sys.stderr)
        ok = False
    if world > 1 and peers is not None:
        # sanity check of the peer path (every rank takes part): the summed
        # grad_X must be bit-identical on every rank
        gxs = [torch.empty_like(gx) for _ in range(world)]
        dist.all_gather(gxs, gx)
        if not all(torch.equal(g_, gxs[0]) for g_ in gxs[1:]):
            print("peer all-reduce gave different grad_X across ranks; using NCCL", file=sys.stderr)
            ok = False
        # every rank must agree before the timed region (and on the path taken)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            head.peers = None
            gx_allreduce[0] = "nccl all_reduce (peer path failed in warm-up)"
            for s in range(a.warmup):
                step_fn(s, batch_dev, gx)
    torch.cuda.synchronize()

    # ---------------- timed region (device-resident inputs)
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local)
    _lib.profile_read()
    _lib.profile_clock()
    _lib.profile_enable(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    if clocks.nvml is None:
        time.sleep(0.3)   # nvidia-smi needs to be running before the timed region
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s in range(a.steps):
        step_fn(a.warmup + s, batch_dev, gx)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    _lib.profile_enable(False)
    ms_fwd, n_fwd, ms_bwd, n_bwd = _lib.profile_read()
    # effective SM clock inside the kernels (block 0's clock64 / globaltimer):
    # NVML's clock reading lags; the heavy kernels run power-limited below it
    kclk = _lib.profile_clock()
    clk["kernel_mhz"] = {k: (round(v, 1) if v else None) for k, v in kclk.items()}
    t_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    peak_mem = torch.cuda.max_memory_allocated(dev) - mem0 + W.numel() * W.element_size()
    if head.comp is not None:   # allocated with the head, before mem0
        peak_mem += head.comp.numel() * head.comp.element_size()
    _lib.check(_lib.load().xmc_head_check(head.handle(a.batch, len(si)).h, _lib.stream_ptr()))

    # ---------------- end-to-end through the public API, host buffers
    Xp = torch.from_numpy(Xh).pin_memory()
    sip = torch.from_numpy(si.astype(np.int32)).pin_memory()
    lip = torch.from_numpy(li.astype(np.int32)).pin_memory()
    gxh = torch.empty((a.batch, a.dim), dtype=torch.float32).pin_memory()
    Xe = torch.empty_like(Xd)
    sie = torch.empty_like(sid)
    lie = torch.empty_like(lid)
    from paper_2510_11168_b200.parallel import broadcast_batch

    def e2e_step(s):
        if world > 1:
            # rank 0 holds the batch (pinned host X + global positives): H2D
            # on rank 0, broadcast to every rank (SURVEY 8(e) X broadcast)
            broadcast_batch(Xp, sip, lip, src=0, out=(Xe, sie, lie))
        else:
            Xe.copy_(Xp, non_blocking=True)
            sie.copy_(sip, non_blocking=True)
            lie.copy_(lip, non_blocking=True)
        r = step_fn(s, xmc.BatchInput(Xe, sie, lie), gx)
        gxh.copy_(r, non_blocking=True)
        stream.synchronize()

    for s in range(3):   # warm-up of the host path (pinned copies, first-call costs)
        e2e_step(9_000 + s)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(a.e2e_steps):
        e2e_step(10_000 + s)
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item()) / a.e2e_steps

    # ---------------- the reference-precision mode on the same workload
    ref_prec = None
    if a.ref_steps > 0 and a.precision == "operand":
        head.precision = "reference"
        for s in range(2):
            step_fn(20_000 + s, batch_dev, gx)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        r0_, r1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0_.record(stream)
        for s in range(a.ref_steps):
            step_fn(20_100 + s, batch_dev, gx)
        r1_.record(stream)
        torch.cuda.synchronize()
        tr_ = torch.tensor([r0_.elapsed_time(r1_)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tr_, op=dist.ReduceOp.MAX)
        ms_ref = float(tr_.item()) / a.ref_steps
        _lib.check(_lib.load().xmc_head_check(head.handle(a.batch, len(si)).h, _lib.stream_ptr()))
        ref_prec = {"value": a.batch / (ms_ref * 1e-3), "unit": "samples/s", "ms_per_step": ms_ref,
                    "steps": a.ref_steps,
                    "what": "same step with ChunkedHead(precision='reference'): the reference's fp32 G as three "
                            "exact bf16 planes, kind::f16 backward GEMMs (device-resident inputs)"}
        head.precision = a.precision

    # ---------------- the bf16-G operand mode (FP8 weights, BF16 logit
    # gradients as in the paper; e4m3 heads) on the same workload
    bf16g = None
    if a.bf16g_steps > 0 and world == 1 and a.fmt == "e4m3" and a.precision == "operand" \
            and a.g_format != "bf16" and a.batch <= 256 and not a.kahan:
        hg = xmc.ChunkedHead(xmc.QuantizedMatrix(W, fmt), num_chunks=a.chunks, num_labels_global=a.labels,
                             label_offset=lo, precision="operand", g_format="bf16")
        for s in range(2):
            xmc.head_update(hg, batch_dev, cfg, rng, 30_000 + s, grad_out=gx, check=False)
        torch.cuda.synchronize()
        b0_, b1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0_.record(stream)
        for s in range(a.bf16g_steps):
            xmc.head_update(hg, batch_dev, cfg, rng, 30_100 + s, grad_out=gx, check=False)
        b1_.record(stream)
        torch.cuda.synchronize()
        ms_b = b0_.elapsed_time(b1_) / a.bf16g_steps
        _lib.check(_lib.load().xmc_head_check(hg.handle(a.batch, len(si)).h, _lib.stream_ptr()))
        bf16g = {"value": a.batch / (ms_b * 1e-3), "unit": "samples/s", "ms_per_step": ms_b,
                 "steps": a.bf16g_steps,
                 "what": "same step with ChunkedHead(precision='operand', g_format='bf16'): FP8 weights with BF16 "
                         "logit gradients (the paper's Algorithm 1), kind::f16 backward GEMMs on bf16 operand "
                         "tiles (device-resident inputs)"}
        del hg

    # ---------------- roofline of the dominant kernel
    peaks = load_peaks()
    L_r, B, D = hi - lo, a.batch, a.dim
    eb = 1 if a.fmt == "e4m3" else 2
    Bp = 128 if (eb == 1 and B <= 128) else (256 if eb == 1 else max(64, 1 << (B - 1).bit_length()))
    per_step = {"fwd": (ms_fwd / max(a.steps, 1), n_fwd // max(a.steps, 1)),
                "bwd": (ms_bwd / max(a.steps, 1), n_bwd // max(a.steps, 1))}
    dom = "bwd" if ms_bwd >= ms_fwd else "fwd"
    n_launch = max(per_step[dom][1], 1)
    ms_launch = per_step[dom][0] / n_launch
    rows_launch = L_r / n_launch
    # algorithmic work per launch: flops of its GEMMs and the
    # bytes of W it must move (bwd: read + write, fwd: read); the G buffer
    # round trip is a design cost, reported separately as design_bytes
    gb = 1 if eb == 1 else 2
    if dom == "bwd":   # grad_X + dW GEMMs, W read+write
        flops = 4.0 * B * rows_launch * D
        bytes_ = 2.0 * rows_launch * D * eb
        design = bytes_ + rows_launch * Bp * gb
    else:              # logits GEMM, W read
        flops = 2.0 * B * rows_launch * D
        bytes_ = rows_launch * D * eb
        design = bytes_ + rows_launch * Bp * gb
    # Burst vs sustained peak by the clocks seen in the timed region: a short
    # region runs at boost clocks (burst peak); a long one hits the ~1 kW power
    # cap, the SM clock drops to ~1.3-1.4 GHz and the sustained peak applies.
    smax = clk.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    burst = bool(clk.get("sm_mhz")) and clk["sm_mhz"] >= 0.95 * smax and "sw_power_cap" not in clk.get("reasons", [])
    regime = "burst" if burst else "sustained"
    # Tensor peak = the tensor pipe's measured issue rate (tools/probe_mma.cu,
    # profiles/r1_probe_mma.txt: kind::f8f6f4 16384 flop/clk/SM, kind::f16 8192,
    # for N >= 128 in either majorness) x SMs x the SM clock seen in the timed
    # region.  This is the hardware ceiling (4.77 PF fp8 at 1965 MHz, 4.4-4.5 PF
    # at the ~1.84 GHz a dense MMA loop holds); cuBLAS-class library GEMMs reach
    # less (torch._scaled_mm 8192^3: 3.1 PF, profiles/fp8_peak.json).
    # the clock the dominant kernel actually ran at (in-kernel clock64 /
    # globaltimer), else NVML's reading
    sm_mhz = (clk.get("kernel_mhz") or {}).get(dom) or clk.get("sm_mhz") or smax
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    tc_peak = (16384.0 if eb == 1 else 8192.0) * n_sms * sm_mhz * 1e6 / 1e12
    tc_src = (f"tensor pipe {'16384' if eb == 1 else '8192'} flop/clk/SM (probe_mma) x {n_sms} SMs x "
              f"{sm_mhz:.0f} MHz in-kernel clock ({regime})")
    t_tc = flops / (tc_peak * 1e12)
    t_hbm = bytes_ / (peaks["hbm_gbs"] * 1e9)
    bound = "tensor" if t_tc >= t_hbm else "hbm"
    if bound == "tensor":
        achieved = flops / (ms_launch * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                "frac": achieved / tc_peak}
    else:
        achieved = bytes_ / (ms_launch * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"]}
    # DRAM traffic of the same kernel from the committed ncu capture (per launch,
    # scaled to this launch's rows): profiles/ncu_traffic.json
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(dom)
        if tr and tr.get("fmt") == a.fmt and tr.get("batch") == B:
            traffic = tr["dram_bytes"] * rows_launch / tr["rows"]
    roof.update({"kernel": "xmc_bwd_kernel (grad_X + dW + SGD/SR update)" if dom == "bwd"
                 else "xmc_fwd_kernel (logits + sigmoid - Y)", "traffic": traffic,
                 "ms_per_launch": ms_launch, "launches_per_step": n_launch,
                 "algorithmic_flops_per_launch": flops, "algorithmic_bytes_per_launch": bytes_,
                 "design_bytes_per_launch": design,
                 "tensor_frac_of_nominal": (flops / (ms_launch * 1e-3) / 1e12) / (4500.0 if eb == 1 else 2250.0),
                 "hbm_frac": (bytes_ / (ms_launch * 1e-3) / 1e9) / peaks["hbm_gbs"],
                 "peak_source": tc_src if bound == "tensor" else f"hbm {peaks['source']}",
                 "peak_regime": regime,
                 "step_kernel_ms": {"fwd": per_step["fwd"][0], "bwd": per_step["bwd"][0]}})
    step_flops = 6.0 * B * a.labels * D
    ms_step = t_ms / a.steps
    value = B * a.steps / (t_ms * 1e-3)
    out = {"metric": metric, "value": value, "unit": "samples/s", "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": a.fmt, "data": "synthetic", "config": config,
           "e2e": {"value": B / (e2e_ms * 1e-3), "unit": "samples/s",
                   "h2d_bytes_per_step": int(Xh.nbytes + 8 * len(si)),
                   "d2h_bytes_per_step": int(B * D * 4), "ms_per_step": e2e_ms},
           "roofline": roof,
           "grad_x_allreduce": gx_allreduce[0],
           "reference_precision": ref_prec,
           "bf16_g_precision": bf16g,
           "step_tflops": step_flops / (ms_step * 1e-3) / 1e12,
           # against dense FP8 at B200's nominal 4.5 PF and the measured
           # torch._scaled_mm FP8 GEMM (profiles/fp8_peak.json, burst)
           "step_frac_of_nominal_fp8": (step_flops / (ms_step * 1e-3) / 1e12 / (4500.0 * world)
                                        if eb == 1 else None),
           "step_frac_of_measured_fp8_gemm": (step_flops / (ms_step * 1e-3) / 1e12 / (fp8_gemm_peak() * world)
                                              if eb == 1 and fp8_gemm_peak() else None),
           "step_frac_of_tc_peak": step_flops / (ms_step * 1e-3) / 1e12 / (tc_peak * world),
           "peak_hbm_gib_per_gpu": peak_mem / 2**30,
           # our kernels in the timed region: every fwd / bwd launch (counted by the
           # library's profiler) + per step: x_prep fused with single-CTA bucketing
           # for <= 12,288 positives, else x_prep fused with counting + scan +
           # scatter; and the grad_X reduce (peer all-reduce kernel for N > 1)
           "gpu_launches": int(n_fwd + n_bwd + a.steps * ((1 if len(si) <= 12288 else 3) + 1)),
           "clocks": clk}
    if rank == 0 and world == 1 and not a.no_cpu:
        cb = cpu_baseline(a, a.cpu_seconds)
        out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
