#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a per-kernel
table (launches, total device time, share):

    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/<round>_launches_summary.txt

The launches are cold-cache and serialised (ncu replays each one alone), so compare SHARES
with the bench's live per-launch CUDA-event table, not absolute times."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    col = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[col["Metric Value"]].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[col["Metric Unit"]], 1.0)
        a = agg[r[col["Kernel Name"]].split("(")[0]]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.1f} ms of kernel time (ncu, serialised)")
    print("# kernel | launches | total ms | share %")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k} | {v[0]} | {v[1] / 1e3:.2f} | {100 * v[1] / tot:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
