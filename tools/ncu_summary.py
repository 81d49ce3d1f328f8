"""Summarise an `ncu --set full` report into profiles/ (tools only).

    python tools/ncu_summary.py gpurun_out/<report>.ncu-rep profiles/<round>_ncu_full_summary.csv

Writes the per-launch CSV summary (duration, DRAM bytes, throughput, grid,
registers, stall ratios) and updates profiles/ncu_traffic.json, the per-kernel
DRAM traffic that bench.py reports as roofline.traffic (dram__bytes_read.sum +
dram__bytes_write.sum per launch, averaged over the captured launches).
"""
import csv
import io
import json
import os
import subprocess
import sys

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
COLS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main(rep: str, out_csv: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, body = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    name_i = idx["Kernel Name"]
    per = {}
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + [c + (f" ({units[idx[c]]})" if c in idx and units[idx[c]] else "")
                                 for c in COLS if c in idx])
        for r in body:
            k = r[name_i].split("(")[0].replace("smoe::", "")
            w.writerow([k] + [r[idx[c]] for c in COLS if c in idx])

            def val(c):
                return float(r[idx[c]].replace(",", "")) * UNITS.get(units[idx[c]], 1.0)
            d = per.setdefault(k, {"n": 0, "rd": 0.0, "wr": 0.0, "us": 0.0})
            d["n"] += 1
            d["rd"] += val("dram__bytes_read.sum")
            d["wr"] += val("dram__bytes_write.sum")
            d["us"] += float(r[idx["gpu__time_duration.sum"]])
    tj = os.path.join(os.path.dirname(out_csv), "ncu_traffic.json")
    try:
        cur = json.load(open(tj))
    except Exception:
        cur = {"kernels": {}}
    for k, d in per.items():
        cur["kernels"][k] = {"dram_read_bytes": d["rd"] / d["n"], "dram_write_bytes": d["wr"] / d["n"],
                             "duration_us_cold": d["us"] / d["n"], "launches": d["n"],
                             "report": os.path.basename(rep)}
    cur["how"] = ("ncu --set full --clock-control none --import-source on (one GPU, cold, "
                  "serialised launches); bytes per launch averaged over the captured launches")
    json.dump(cur, open(tj, "w"), indent=1, sort_keys=True)
    print(json.dumps(cur["kernels"], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
