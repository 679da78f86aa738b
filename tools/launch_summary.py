"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals.

    python tools/launch_summary.py launches.csv [--last-fraction 0.5]
"""
import collections
import csv
import re
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[1:]:
        if len(r) != len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[idx["Kernel Name"]]).replace("<unnamed>::", "")
        v = float(r[idx["Metric Value"]])
        unit = r[idx["Metric Unit"]]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        out.append((name, v, r[idx["Grid Size"]]))
    return out


def main():
    path = sys.argv[1]
    frac = float(sys.argv[sys.argv.index("--last-fraction") + 1]) if "--last-fraction" in sys.argv else 0.5
    data = load(path)
    data = data[int(len(data) * (1 - frac)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, v, _ in data:
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"launches {len(data)}  total {tot:.1f} us (serialised, cold-cache)")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:34s} n={v[0]:5d} us={v[1]:10.1f} ({100 * v[1] / tot:5.1f}%) avg={v[1] / v[0]:8.1f}")


if __name__ == "__main__":
    main()
