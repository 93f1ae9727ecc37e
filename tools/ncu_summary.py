#!/usr/bin/env python3
"""Summarise an ncu --set full report of the DFS kernel (the evidence the north star
asks for): shared-memory bank conflicts and wavefronts, ALU / FMA pipe utilisation,
issue activity, occupancy, SIMT efficiency, stall mix, DRAM traffic.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [> profiles/xxx.md]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "kernel time"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block"),
    ("launch__occupancy_limit_shared_mem", "blocks/SM limit (smem)"),
    ("launch__occupancy_limit_registers", "blocks/SM limit (regs)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads / warp instruction (SIMT eff. x32)"),
    ("sm__inst_executed.avg.per_cycle_active", "warp inst / cycle / SM (max 4)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy pipe % (IMAD)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem st wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        print(f"### {d.get('Kernel Name', ('?',))[0][:100]}\n")
        print("| metric | value | ncu name |\n|---|---|---|")
        for k, label in KEYS:
            if k in d:
                v, u = d[k]
                print(f"| {label} | {v} {u} | `{k}` |")
        stalls = []
        for h in hdr:
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(d[h][0])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        print("\nStall reasons (warps per issue-active cycle, >= 0.05): " +
              ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)) + "\n")


if __name__ == "__main__":
    main()
