"""Summarise an ncu --set full report (raw page) into the figures DESIGN.md
and bench.py's roofline.traffic cite.  Usage: python ncu_summary.py rep..."""
import csv
import json
import subprocess
import sys

KEYS = {
    "kernel": "Kernel Name",
    "time_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_dyn": "launch__shared_mem_per_block_dynamic",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for k, name in KEYS.items():
        if name in head:
            i = head.index(name)
            v = vals[i]
            try:
                v = float(v.replace(",", "")) * SCALE.get(units[i], 1)
            except ValueError:
                pass
            res[k] = v
    stalls = []
    for i, name in enumerate(head):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((round(float(vals[i]), 2), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    res["top_stalls"] = sorted(stalls, reverse=True)[:5]
    res["dram_bytes"] = res.get("dram_read", 0) + res.get("dram_write", 0)
    return res


if __name__ == "__main__":
    print(json.dumps({r: summarise(r) for r in sys.argv[1:]}, indent=1))
