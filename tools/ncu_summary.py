#!/usr/bin/env python3
"""Summarise an `ncu --set full` capture (read here with `ncu -i ... --page raw --csv`)
into profiles/: one markdown table of the key per-launch metrics and a JSON
file bench.py reads for `roofline.traffic` (dram read+write bytes per launch).

    python tools/ncu_summary.py gpurun_out/filter_tc.ncu-rep profiles/r01_filter_tc_ncu [kernel-regex]
"""
import re
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__cycles_elapsed.avg.per_second", "SM clk"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 rd sectors"),
    ("lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * scale


def main(rep, out_prefix, pattern=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    cols = [(hdr.index(m), m, label) for m, label in METRICS if m in hdr]
    lines = ["| # | kernel | " + " | ".join(f"{label} ({units[i]})" for i, _, label in cols) + " |",
             "|---|---|" + "---|" * len(cols)]
    per_launch = []
    if pattern:
        data = [r for r in data if re.search(pattern, r[ki])]
    for n, r in enumerate(data):
        lines.append(f"| {n} | `{r[ki][:60]}` | " + " | ".join(r[i] for i, _, _ in cols) + " |")
        rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        t_ms = float(r[hdr.index("gpu__time_duration.sum")]) * (1e-3 if units[hdr.index("gpu__time_duration.sum")] == "us" else 1)
        per_launch.append({"kernel": r[ki], "dram_bytes": rd + wr, "ms": t_ms})
    with open(out_prefix + ".md", "w") as f:
        f.write(f"ncu --set full --clock-control none capture: `{rep}`\n\n" + "\n".join(lines) + "\n")
    summary = {"source": rep, "launches": per_launch,
               "mean_dram_bytes_per_launch": sum(x["dram_bytes"] for x in per_launch) / max(1, len(per_launch))}
    with open(out_prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
