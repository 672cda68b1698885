"""Compact summary of an ncu --set full report: duration, DRAM bytes and
throughput, tensor-pipe / L2 / SM utilisation, top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/prof_bwd.ncu-rep [--json out.json]
"""

import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    # tensor pipe: sm__pipe_tensor_cycles_active (SM clock domain) is the one that
    # equals the flop-derived utilisation (flops / (16384 flop/clk/SM fp8 x SMs x
    # SM clock x duration)); the *_realtime variant counts in another clock domain
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_realtime_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "dram_TBps": "dram__bytes.sum.per_second",
    "smem_lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "inst_executed": "smsp__inst_executed.sum",
    "tensor_mem_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
    "sm_clock_mhz": "sm__cycles_elapsed.avg.per_second",
}


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:80]}
        for k, m in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u == "Gbyte":
                    v *= 1000.0
                elif u == "Kbyte":
                    v /= 1000.0
                elif u == "byte":
                    v /= 1e6
                elif u in ("msecond", "ms") and k == "duration_us":
                    v *= 1000.0
                elif u in ("nsecond", "ns") and k == "duration_us":
                    v /= 1000.0
                elif u in ("second", "s") and k == "duration_us":
                    v *= 1e6
                if k == "dram_TBps":
                    v = v if u == "Tbyte/s" else (v / 1000.0 if u == "Gbyte/s" else v)
                if k == "sm_clock_mhz":
                    v = v / 1e6 if u in ("cycle/second", "") else v * (1000.0 if u.startswith("G") else 1.0)
                d[k] = round(v, 3)
        stalls = {}
        for i, n in enumerate(hdr):
            if n.startswith("smsp__average_warp_latency_issue_stalled_") and n.endswith(".pct"):
                pass
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in
                               sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        # the exact ncu metric behind every key (the tensor-pipe figure is
        # tensor_pipe_pct = sm__pipe_tensor_cycles_active; tensor_mem_pct is the
        # tensor core's shared/tensor-memory traffic, not its math pipe)
        d["metrics"] = {k: m for k, m in KEYS.items() if k in d}
        out.append(d)
    return out


def reconcile(d, flops, per_clk):
    """flop-derived tensor utilisation next to the ncu metric"""
    if "duration_us" in d and "sm_clock_mhz" in d:
        peak = per_clk * 148 * d["sm_clock_mhz"] * 1e6
        d["algorithmic_flops"] = flops
        d["flop_derived_tensor_pct"] = round(100.0 * flops / (d["duration_us"] * 1e-6) / peak, 1)
        d["flop_peak_note"] = f"{per_clk} flop/clk/SM x 148 SMs x {d['sm_clock_mhz']:.0f} MHz"


if __name__ == "__main__":
    res = summarize(sys.argv[1])
    if "--flops" in sys.argv:
        fl = float(sys.argv[sys.argv.index("--flops") + 1])
        pc = float(sys.argv[sys.argv.index("--per-clk") + 1]) if "--per-clk" in sys.argv else 16384.0
        for d in res:
            reconcile(d, fl, pc)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
    for d in res:
        print(json.dumps(d))
