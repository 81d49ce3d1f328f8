"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list (tools only).

    python tools/launch_summary.py gpurun_out/launches.csv profiles/<round>_launches_summary.csv [exclude-regex]

Per kernel: launches, total and average ns, and share of the summed GPU time
(ncu serialises launches and runs them cold: compare shares, not absolutes).
"""
import csv
import re
import sys
from collections import defaultdict


def main(src: str, dst: str, exclude: str = "") -> None:
    rows = [r for r in csv.reader(open(src)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("smoe::", "")
        if exclude and re.search(exclude, name):
            continue
        scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    all_ns = sum(tot.values())
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_ns", "avg_ns", "share_of_gpu_time"])
        for k in sorted(tot, key=lambda k: -tot[k]):
            w.writerow([k, cnt[k], int(tot[k]), int(tot[k] / cnt[k]), f"{tot[k] / all_ns:.4f}"])
    print(open(dst).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
