#!/usr/bin/env python
"""Per-kernel means of the memory-pipeline metrics of an `ncu --set full` raw CSV
(`ncu -i rep --page raw --csv > raw.csv`), written as a text table for profiles/:

    python scripts/ncu_metrics.py gpurun_out/r4f_raw.csv profiles/r4f_ncu_metrics_C4_Aside.txt "title"
"""
import collections
import csv
import re
import sys

METRICS = [
    ("us", "gpu__time_duration.sum"),
    ("dram_rd_GB", "dram__bytes_read.sum"),
    ("dram_wr_GB", "dram__bytes_write.sum"),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l1tex_%", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("lts_%", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l1_hit_%", "l1tex__t_sector_hit_rate.pct"),
    ("l2_hit_%", "lts__t_sector_hit_rate.pct"),
    ("ld_req_M", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    ("ld_sect_M", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    ("l2_rd_sect_M", "lts__t_sectors_srcunit_tex_op_read.sum"),
    ("warps_act_%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue_act_%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("stall_long_sb", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
    ("regs", "launch__registers_per_thread"),
]
SCALE = {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "ms": 1e3, "us": 1.0, "ns": 1e-3}


def main(raw, out, title=""):
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).replace("void ", "").strip()
        d = agg.setdefault(name, collections.defaultdict(list))
        for short, m in METRICS:
            if m not in col:
                continue
            try:
                v = float(r[col[m]].replace(",", ""))
            except ValueError:
                continue
            u = units[col[m]]
            if short.endswith("_M"):
                v *= 1e-6
            elif u in SCALE:
                v *= SCALE[u]
            d[short].append(v)
    lines = [f"# {title}", "# per-kernel means over the profiled launches (ncu --set full --clock-control none); "
             "DRAM in GB per launch, requests/sectors in millions per launch",
             "kernel | launches | " + " | ".join(s for s, _ in METRICS)]
    for name, d in agg.items():
        n = len(d["us"])
        lines.append(f"{name} | {n} | " + " | ".join(
            (f"{sum(d[s]) / len(d[s]):.3g}" if d[s] else "-") for s, _ in METRICS))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
