#!/usr/bin/env python
"""Summarise an ncu --set full report into profiles/ncu_<name>.json.

  python tools/ncu_summary.py gpurun_out/prof_cfg2.ncu-rep cfg2

Keeps the metrics the roofline in bench.py and DESIGN.md cite: duration,
DRAM bytes (read + write = `traffic`), L2/xbar bytes, tensor-pipe and SM
utilisation, occupancy and registers.
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]

UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
        "s": 1.0}


def main(rep, name, out_dir="profiles"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                scale = UNIT.get(units[i], 1.0)
                rec[k] = v * scale if units[i] in UNIT else v
        launches.append(rec)
    first = launches[0] if launches else {}
    summary = {
        "report": os.path.basename(rep), "workload": name,
        "kernel": first.get("kernel"),
        "duration_s": first.get("gpu__time_duration.sum"),
        "dram_bytes_per_launch": (first.get("dram__bytes_read.sum", 0) +
                                  first.get("dram__bytes_write.sum", 0)) or None,
        "note": "ncu --set full --clock-control none; cold caches and serialised replays: "
                "compare shares, not absolute times",
        "launches": launches,
    }
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, f"ncu_{name}.json")
    with open(path, "w") as f:
        json.dump(summary, f, indent=1)
    print(path, json.dumps({k: v for k, v in summary.items() if k != "launches"}))


if __name__ == "__main__":
    main(*sys.argv[1:])
