"""Summarise ncu captures into the JSON files kept under profiles/.

    python profiles/summarize_ncu.py full  OUT.json  REP.ncu-rep [REP2.ncu-rep ...]
        per-kernel key metrics of `ncu --set full` reports (one entry per profiled launch)
    python profiles/summarize_ncu.py traffic OUT.json REP.ncu-rep [...]
        per-kernel DRAM bytes per launch (read + write), the `roofline.traffic` source of bench.py

Reads the reports with `ncu -i REP --page raw --csv` (this container has ncu; no GPU needed).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw_rows(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def short(name: str) -> str:
    for k in ("k_extract", "k_rebuild", "k_ematch", "k_join"):
        if k in name:
            return k[2:]
    return name


def main() -> None:
    mode, out, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    rows = [r for rep in reps for r in raw_rows(rep)]
    if mode == "full":
        res = []
        for d in rows:
            e = {k: d[k][0] for k in ("Kernel Name", "Grid Size", "Block Size") if k in d}
            for m in METRICS:
                if m in d:
                    v, u = d[m]
                    e[m] = f"{v} {u}".strip()
            res.append(e)
    else:
        res = {}
        for d in rows:
            b = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, u = d[m]
                b += float(v.replace(",", "")) * SCALE.get(u, 1)
            res.setdefault(short(d["Kernel Name"][0]), b)
        res["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full, "
                        "4096 NasRNN leaves (" + ", ".join(reps) + ")")
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
        fh.write("\n")


if __name__ == "__main__":
    main()
