#!/usr/bin/env python
"""Build profiles/ncu_summary.json (read by bench.py for roofline.traffic) from the
committed per-kernel ncu summaries (tools/ncu_extract.py output).

    python tools/make_ncu_summary.py KERNEL:CONFIG:profiles/FILE.json ...
"""
import json
import sys

out = {}
for arg in sys.argv[1:]:
    kernel, config, path = arg.split(":", 2)
    k = json.load(open(path))["kernels"][0]
    out.setdefault(kernel, {})[config] = {
        "dram_bytes_per_launch": k["dram_bytes_per_launch"],
        "gpu_time_s": k["gpu__time_duration.sum"],
        "dram_pct_peak": k["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
        "issue_active_pct": k["smsp__issue_active.avg.pct_of_peak_sustained_active"],
        "pipe_alu_pct": k.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "pipe_fma_pct": k.get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "source": path,
    }
json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
