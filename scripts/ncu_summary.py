#!/usr/bin/env python
"""Summarise ncu --set full captures into profiles/ (text) and the per-kernel
DRAM traffic table profiles/ncu_traffic.json that bench.py reports as
roofline.traffic (dram__bytes_read.sum + dram__bytes_write.sum per launch,
divided by the streams one launch processes).

usage: scripts/ncu_summary.py <tag> <rep or raw csv> <streams> <layer key ("<config>/L<i>[/raw]")> [...]
       (one name per captured launch, in launch order)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    """The raw metrics page: from a report, or from its saved CSV (ncu -i rep --page raw --csv)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    tag, rep, streams = sys.argv[1], sys.argv[2], int(sys.argv[3])
    names = sys.argv[4:]
    h, units, rows = raw(rep)
    lines = [f"ncu --set full --clock-control none ({os.path.basename(rep)}), {streams} streams per launch"]
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for i, r in enumerate(rows):
        name = names[i] if i < len(names) else r[h.index("Kernel Name")][:80]
        lines.append(f"--- launch {i}: {name}")
        vals = {}
        for k in KEYS:
            if k in h:
                j = h.index(k)
                vals[k] = (r[j], units[j])
                lines.append(f"  {k} [{units[j]}] = {r[j]}")
        rd = float(vals["dram__bytes_read.sum"][0]) * SCALE[vals["dram__bytes_read.sum"][1]]
        wr = float(vals["dram__bytes_write.sum"][0]) * SCALE[vals["dram__bytes_write.sum"][1]]
        lines.append(f"  traffic (read+write) = {(rd + wr) / 1e6:.1f} MB per launch, {(rd + wr) / streams / 1e6:.4f} MB per stream-step")
        traffic[name] = {"bytes_per_stream_step": (rd + wr) / streams, "source": os.path.basename(rep), "tag": tag}
    with open(os.path.join(ROOT, "profiles", f"{tag}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
