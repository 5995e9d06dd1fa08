"""Summarise an ncu report (--set full) per kernel: time, DRAM bytes, pipe/issue stats.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cycles_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "launch__registers_per_thread": "regs",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "thread_dfma",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "thread_dmul",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "thread_dadd",
    "smsp__warps_active.avg.per_cycle_active": "warps_per_smsp",
    "smsp__average_warp_latency_issue_stalled_barrier": "stall_barrier",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_sb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_sb",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio": "stall_math",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "stall_mio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio": "stall_lg",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio": "stall_membar",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio": "stall_drain",
}


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]}
        for k, name in WANT.items():
            if k in hdr:
                v = r[hdr.index(k)]
                u = units[hdr.index(k)]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                if u == "ms" and isinstance(v, float):
                    v *= 1000.0
                    u = "us"
                if u == "Mbyte" and isinstance(v, float):
                    v /= 1000.0
                    u = "Gbyte"
                if u == "Kbyte" and isinstance(v, float):
                    v /= 1e6
                    u = "Gbyte"
                if u == "byte" and isinstance(v, float):
                    v /= 1e9
                    u = "Gbyte"
                d[name] = v
                if name == "time":
                    d["time_unit"] = u
        out.append(d)
    return out


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    for d in res:
        print(" | ".join(f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}" for k, v in d.items()))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
