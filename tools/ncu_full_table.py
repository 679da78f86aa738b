"""Table of the key `ncu --set full` metrics per captured launch (from `ncu -i rep --page raw --csv`).

    ncu -i gpurun_out/full.ncu-rep --page raw --csv > raw.csv; python tools/ncu_full_table.py raw.csv
"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
col = {k: i for i, k in enumerate(h)}
want = [("dur_us", "gpu__time_duration.sum", 1e-3), ("grid", "launch__grid_size", 1), ("block", "launch__block_size", 1),
        ("regs", "launch__registers_per_thread", 1),
        ("occ_ach%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
        ("dmma%act", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
        ("sm_thru%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
        ("dramR_MB", "dram__bytes_read.sum", 1), ("dramW_MB", "dram__bytes_write.sum", 1),
        ("L2hit%", "lts__t_sector_hit_rate.pct", 1)]
print("kernel | " + " | ".join(w[0] for w in want) + " | dram_GB/s")
for r in rows[2:]:
    nm = re.sub(r"\(anonymous namespace\)::|<unnamed>::|^void ", "", r[col["Kernel Name"]]).split("(")[0]
    vals = []
    for name, key, _ in want:
        if key not in col:
            vals.append("-")
            continue
        v, u = r[col[key]].replace(",", ""), units[col[key]]
        try:
            x = float(v)
        except ValueError:
            vals.append(v)
            continue
        if name == "dur_us":
            x = x * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}.get(u, 1)
        elif name in ("dramR_MB", "dramW_MB"):
            x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
        vals.append(f"{x:.4g}")
    try:
        gbs = (float(vals[7]) + float(vals[8])) / float(vals[0]) * 1e3  # MB/us -> GB/s
    except (ValueError, ZeroDivisionError):
        gbs = float("nan")
    print(nm + " | " + " | ".join(vals) + f" | {gbs:.0f}")
