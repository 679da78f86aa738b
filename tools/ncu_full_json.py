"""Per-kernel JSON of `ncu --set full` captures (raw-page CSV exports, optionally gzipped): duration, DRAM bytes,
FP64 tensor (DMMA) pipe activity, occupancy, registers.  bench.py reads `dram_bytes_per_launch` of the dominant kind.

    python tools/ncu_full_json.py profiles/r02_ncu_kernels.json gpurun_out/n_full_*.raw.csv.gz
"""
import csv
import gzip
import io
import json
import re
import sys

KINDS = {4: "trail_kernel", 8: "tgemm_kernel", 9: "rgemm_kernel", 11: "schur_kernel"}
M = {"dur": "gpu__time_duration.sum", "dr": "dram__bytes_read.sum", "dw": "dram__bytes_write.sum",
     "dmma": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
     "fp64": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
     "occ": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread",
     "grid": "launch__grid_size", "l2hit": "lts__t_sector_hit_rate.pct"}
U = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for path in sys.argv[2:]:
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}
    for r in rows[2:]:
        nm = r[col["Kernel Name"]]
        m = re.search(r"tile_tma_kernel(?:ILi|<)(\d+)", nm)
        if m:
            name = KINDS.get(int(m.group(1)), nm)
        else:
            m = re.search(r"([a-z_0-9]+_kernel)", nm)
            name = m.group(1) if m else nm[:40]

        def val(key):
            if M[key] not in col:
                return None
            try:
                return float(r[col[M[key]]].replace(",", "")) * U.get(units[col[M[key]]], 1)
            except ValueError:
                return None

        d = out.setdefault(name, {"launches": 0, "seconds": 0.0, "dram_bytes": 0.0, "samples": []})
        d["launches"] += 1
        d["seconds"] += val("dur") or 0.0
        d["dram_bytes"] += (val("dr") or 0.0) + (val("dw") or 0.0)
        d["samples"].append({"capture": path.split("/")[-1], "us": round((val("dur") or 0) * 1e6, 1),
                             "dram_MB": round(((val("dr") or 0) + (val("dw") or 0)) / 1e6, 2),
                             "dmma_pipe_pct": val("dmma"), "fp64_pipe_pct": val("fp64"), "occupancy_pct": val("occ"),
                             "registers": val("regs"), "grid": val("grid"), "l2_hit_pct": val("l2hit")})
for d in out.values():
    d["dram_bytes_per_launch"] = round(d["dram_bytes"] / max(d["launches"], 1))
    d["dram_GBps"] = round(d["dram_bytes"] / max(d["seconds"], 1e-12) / 1e9, 1)
    d["seconds"] = round(d["seconds"], 6)
    del d["dram_bytes"]
open(sys.argv[1], "w").write(json.dumps(out, indent=1))
for k, d in out.items():
    print(k, d["launches"], "launches", d["dram_bytes_per_launch"] / 1e6, "MB/launch", d["dram_GBps"], "GB/s",
          [s["dmma_pipe_pct"] for s in d["samples"]])
