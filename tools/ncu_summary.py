#!/usr/bin/env python3
"""Summarise an ncu --set full report into profiles/-style JSON: the metrics
the DESIGN / profiles tables quote, per kernel, plus the top stall reasons.

  python tools/ncu_summary.py report.ncu-rep > profiles/rN_step_kernels_ncu.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
        "l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_st.sum"]


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        m = {k: f"{d[k]} {u.get(k, '')}".strip() for k in KEYS if k in d}
        st = {k.split("issue_stalled_")[1].split("_per_issue")[0]: float(d[k])
              for k in hdr if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")}
        tot = sum(st.values()) or 1.0
        m["stall_top"] = {k: round(100 * v / tot, 1)
                          for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]}
        out[name] = m
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
