#!/usr/bin/env python
"""Summarise an ncu report into a small JSON (run where ncu is available).

    python tools/ncu_extract.py REPORT.ncu-rep OUT.json [--label NAME]

Keeps per kernel: duration, DRAM bytes read/written, DRAM throughput %, issue
active %, warps active %, registers, grid/block, smem, instruction count,
pipe utilisations and the warp-stall breakdown (pc sampling).
"""
import csv
import json
import subprocess
import sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__maximum_warps_per_active_cycle_pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__inst_executed_op_shared_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    label = sys.argv[sys.argv.index("--label") + 1] if "--label" in sys.argv else rep
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        k = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for m in KEEP:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in SCALE:
                    v *= SCALE[u]
                    u = "B" if "byte" in u else "s"
                k[m] = v
        st = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        k["stall_pct"] = {a: round(100 * b / tot, 1) for a, b in sorted(st.items(), key=lambda x: -x[1]) if b > 0}
        if "dram__bytes_read.sum" in k and "dram__bytes_write.sum" in k:
            k["dram_bytes_per_launch"] = k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
        kernels.append(k)
    json.dump({"label": label, "kernels": kernels}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
