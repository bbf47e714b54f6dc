"""Merges one ncu metrics capture of a bench winner into
profiles/<round>/ncu_keyed.json, keyed by (workload, tile), which bench.py
reads for roofline.pipe_busy / traffic (tools/capture_keyed.sh runs ncu).

    python tools/ncu_keyed.py <round> <workload> <tile> <ncu.csv> [iterations]

The capture is the launch with the longest gpu__time_duration in the CSV
(--csv --page raw output of one kernel). `iterations` (inner iterations per
launch) adds the FP64 / ALU / FMA warp instructions per 32 iterations.
"""
from __future__ import annotations

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIPES = {"fp64": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
         "alu": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
         "fma": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
         "fmaheavy": "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
         "fp64_cycles": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
         "tensor_cycles": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
         "lsu": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main(rnd, workload, tile, path, iters=None):
    rows = list(csv.reader(open(path)))
    # --page raw --csv: a header row, a units row, then one row per launch
    hdr_i = next(i for i, r in enumerate(rows) if "gpu__time_duration.sum" in r)
    hdr = rows[hdr_i]
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and num(r[hdr.index("gpu__time_duration.sum")])]
    best = max(data, key=lambda r: num(r[hdr.index("gpu__time_duration.sum")]))
    get = lambda m: num(best[hdr.index(m)]) if m in hdr else None  # noqa: E731
    entry = {
        "kernel": best[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None,
        "pipe_pct": {k: get(m) for k, m in PIPES.items() if get(m) is not None},
        "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": get("launch__registers_per_thread"),
        "dram_bytes": (get("dram__bytes_read.sum") or 0) + (get("dram__bytes_write.sum") or 0),
        "duration_ns": get("gpu__time_duration.sum"),
        "capture": os.path.relpath(path, ROOT),
    }
    if iters:
        for pipe in ("fp64", "alu", "fma"):
            n = get(f"sm__inst_executed_pipe_{pipe}.sum")
            if n is not None:
                entry[f"{pipe}_warp_instr_per_32_iters"] = n * 32.0 / float(iters)
    out = os.path.join(ROOT, "profiles", rnd, "ncu_keyed.json")
    d = json.load(open(out)) if os.path.exists(out) else {}
    d.setdefault(workload, {})[tile] = entry
    with open(out, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    print(json.dumps({workload: {tile: entry}}, indent=1))


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1], a[2], a[3], float(a[4]) if len(a) > 4 else None)
