"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,lts__t_bytes.sum --csv) of one solve into per-kernel totals.

    python tools/ncu_summary.py gpurun_out/launches.csv --json profiles/r01_ncu_kernels.json > profiles/r01_ncu_kernels.txt

ncu serialises launches and flushes caches between them: times are cold-cache and
serialised (compare shares, not absolutes); dram bytes are per-launch upper bounds."""
import argparse
import collections
import csv
import json
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--json", default="")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
idx = {k: i for i, k in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
per = {}
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    nm = re.sub(r"\(anonymous namespace\)::|<unnamed>::|^void ", "", r[idx["Kernel Name"]]).split("(")[0]
    m = re.match(r"tile_tma_kernel<\(?(?:int\)?)?(\d+)>", nm) or re.search(r"tile_tma_kernelILi(\d+)E", nm)
    if m:  # the TMA tile engine's four launch kinds (LaunchKind, plan.h): named like the cp.async kernels they replace
        nm = {4: "trail_kernel", 8: "tgemm_kernel", 9: "rgemm_kernel", 11: "schur_kernel"}.get(int(m.group(1)), nm) + "[tma]"
    nm = re.sub(r"<.*", "", nm)
    v = float(r[idx["Metric Value"]].replace(",", "")) * scale.get(r[idx["Metric Unit"]], 1)
    per.setdefault(r[idx["ID"]], {"name": nm})[r[idx["Metric Name"]]] = v
tot = collections.defaultdict(lambda: collections.defaultdict(float))
for d in per.values():
    t = tot[d["name"]]
    t["launches"] += 1
    t["time_s"] += d.get("gpu__time_duration.sum", 0.0)
    t["dram_read"] += d.get("dram__bytes_read.sum", 0.0)
    t["dram_write"] += d.get("dram__bytes_write.sum", 0.0)
    t["l2"] += d.get("lts__t_bytes.sum", 0.0)
T = sum(t["time_s"] for t in tot.values())
print(f"{len(per)} launches, serialized sum {T * 1e3:.2f} ms, dram read "
      f"{sum(t['dram_read'] for t in tot.values()) / 1e9:.2f} GB, write {sum(t['dram_write'] for t in tot.values()) / 1e9:.2f} GB")
out = {}
for nm, t in sorted(tot.items(), key=lambda kv: -kv[1]["time_s"]):
    n = t["launches"]
    out[nm] = {"launches": int(n), "ms": round(t["time_s"] * 1e3, 3), "share": round(t["time_s"] / T, 4),
               "dram_bytes_per_launch": round((t["dram_read"] + t["dram_write"]) / n),
               "l2_bytes_per_launch": round(t["l2"] / n),
               "dram_GBps": round((t["dram_read"] + t["dram_write"]) / max(t["time_s"], 1e-12) / 1e9, 1)}
    print(f"{nm:22s} n={int(n):4d} {t['time_s'] * 1e3:7.2f} ms ({t['time_s'] / T:5.1%})  dram "
          f"{(t['dram_read'] + t['dram_write']) / n / 1e6:7.2f} MB/launch ({out[nm]['dram_GBps']:6.0f} GB/s)  "
          f"L2 {t['l2'] / n / 1e6:7.2f} MB/launch")
for nm in list(out):  # bench.py looks kinds up by their cp.async kernel name
    if nm.endswith("[tma]") and nm[:-5] not in out:
        out[nm[:-5]] = out[nm]
if a.json:
    open(a.json, "w").write(json.dumps(out, indent=1))
