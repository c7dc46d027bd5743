"""Compact per-launch summary of ncu CSV output (for profiles/).

Reads either a `--page raw --csv` export of a report or the stdout of an `ncu --csv
--metrics ...` run (program output lines before the CSV header are skipped) and prints one
JSON object per profiled launch with the metrics that back DESIGN.md's roofline claims:
duration, DRAM bytes, NVLink bytes (when collected), SM / memory throughput, occupancy.

    python tools/ncu_summary.py gpurun_out/r5t_ncu_twoshot4_raw.csv [--algo-bytes B]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "nvltx__bytes.sum": "nvl_tx",
    "nvlrx__bytes.sum": "nvl_rx",
    "nvltx__bytes_data_user.sum": "nvl_tx_user",
    "nvlrx__bytes_data_user.sum": "nvl_rx_user",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def rows_of(text: str):
    lines = text.splitlines()
    start = next((i for i, ln in enumerate(lines) if ln.startswith('"ID"')), None)
    if start is None:
        return None, []
    rd = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    return rd[0], rd[1:]


def num(v: str, unit: str):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(unit, 1.0)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--algo-bytes", type=float, default=0.0, help="algorithmic bytes per launch (adds ratios)")
    a = ap.parse_args()
    text = open(a.path, errors="replace").read()
    head, rows = rows_of(text)
    if head is None:
        sys.exit(f"{a.path}: no ncu CSV header")
    if "Metric Name" in head:  # long format (--metrics ... --csv): one row per metric
        im, iv, iu = head.index("Metric Name"), head.index("Metric Value"), head.index("Metric Unit")
        ik, iid = head.index("Kernel Name"), head.index("ID")
        per: dict = {}
        for r in rows:
            if len(r) <= max(im, iv, iu):
                continue
            d = per.setdefault(r[iid], {"id": int(r[iid]), "kernel": r[ik]})
            if r[im] in KEYS:
                d[KEYS[r[im]]] = num(r[iv], r[iu])
        out = list(per.values())
    else:  # wide raw page: row 0 of the data holds the units
        units, data = rows[0], rows[1:]
        idx = {h: i for i, h in enumerate(head)}
        out = []
        for r in data:
            d = {"id": int(r[idx["ID"]]), "kernel": r[idx["Kernel Name"]]}
            for k, name in KEYS.items():
                if k in idx and r[idx[k]] != "":
                    d[name] = num(r[idx[k]], units[idx[k]])
            out.append(d)
    for d in out:
        if "duration" in d and isinstance(d["duration"], float):
            d["duration_us"] = round(d.pop("duration") * 1e6, 2)
        rd, wr = d.get("dram_read"), d.get("dram_write")
        if isinstance(rd, float) and isinstance(wr, float):
            d["dram_bytes"] = rd + wr
            if d.get("duration_us"):
                d["dram_gbs"] = round((rd + wr) / (d["duration_us"] * 1e-6) / 1e9, 1)
            if a.algo_bytes:
                d["dram_over_algorithmic"] = round((rd + wr) / a.algo_bytes, 3)
        tx = d.get("nvl_tx")
        if isinstance(tx, float) and d.get("duration_us"):
            d["nvl_tx_gbs"] = round(tx / (d["duration_us"] * 1e-6) / 1e9, 1)
        print(json.dumps(d))


if __name__ == "__main__":
    main()
