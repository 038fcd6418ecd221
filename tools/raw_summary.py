#!/usr/bin/env python3
"""Key metrics per kernel from an exported ncu raw page (tools/ncu_export.sh).
usage: tools/raw_summary.py X_raw.csv [kernel-substring]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
want = sys.argv[2] if len(sys.argv) > 2 else ""
for r in rows[2:]:
    name = r[idx["Kernel Name"]]
    if want not in name:
        continue
    print("-" * 72)
    print(name[:150])
    for k in KEYS:
        if k in idx:
            print(f"  {k:82s} {r[idx[k]]:>16s} {units[idx[k]]}")
    st = [(float(r[i] or 0), h) for h, i in idx.items() if h.startswith("smsp__average_warps_issue_stalled_")
          and h.endswith("_per_issue_active.ratio")]
    st.sort(reverse=True)
    print("  top stalls (warps per issue):", ", ".join(f"{h[34:-23]} {v:.2f}" for v, h in st[:6]))
