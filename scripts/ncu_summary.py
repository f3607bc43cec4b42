#!/usr/bin/env python
"""Summarise an `ncu --set full` report into profiles/ (text table + json entries the
bench reads for the roofline `traffic` field):

    python scripts/ncu_summary.py gpurun_out/prof_C2_full.ncu-rep C2 profiles/r1_ncu_full_C2.txt

Per kernel (name without arguments): launches profiled, mean duration, mean DRAM
bytes read+written per launch, DRAM throughput % of peak, achieved occupancy,
registers, L2 hit rate.  Merges {config: {kernel: dram_bytes_per_launch}} into
profiles/ncu_summary.json."""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, config, out_txt):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name, scale=1.0):
        try:
            v = float(r[col[name]].replace(",", ""))
        except (KeyError, ValueError):
            return None
        u = units[col[name]]
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}.get(u, 1.0)
        return v * mult * scale

    agg = collections.OrderedDict()
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[col["Kernel Name"]]).strip()
        d = agg.setdefault(name, collections.defaultdict(list))
        d["us"].append(val(r, "gpu__time_duration.sum"))
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        d["dram"].append((rd or 0) + (wr or 0))
        for k in ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                  "lts__t_sector_hit_rate.pct"):
            d[k].append(val(r, k))
        d["grid"].append(r[col["Grid Size"]])
    mean = lambda xs: sum(x for x in xs if x is not None) / max(1, len([x for x in xs if x is not None]))
    lines = [f"# ncu --set full --clock-control none, config {config}: {rep}",
             "# kernel | launches | mean us | DRAM bytes/launch | DRAM % peak | warps active % | regs | L2 hit % | grids"]
    summary = {}
    for name, d in agg.items():
        lines.append(f"{name} | {len(d['us'])} | {mean(d['us']):.2f} | {mean(d['dram']):.4g} | "
                     f"{mean(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                     f"{mean(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{mean(d['launch__registers_per_thread']):.0f} | {mean(d['lts__t_sector_hit_rate.pct']):.1f} | "
                     f"{sorted(set(d['grid']))[:3]}")
        summary[name] = mean(d["dram"])
    open(out_txt, "w").write("\n".join(lines) + "\n")
    js = os.path.join(ROOT, "profiles", "ncu_summary.json")
    data = json.load(open(js)) if os.path.exists(js) else {}
    data.setdefault("dram_bytes_per_launch", {}).setdefault(config, {}).update(summary)   # merge per kernel
    src = data.setdefault("sources", {}).get(config, [])
    src = src if isinstance(src, list) else [src]
    data["sources"][config] = src + [os.path.basename(out_txt)]
    rnd = os.path.basename(out_txt).split("_")[0]
    data.setdefault("round", {}).update({f"{config}/{k}": rnd for k in summary})
    json.dump(data, open(js, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
