"""Compare two bench --levels captures (per-launch serialized times) kind by kind and group by
group, e.g. the TMA tile engine everywhere vs nowhere, and report the per-kind time each
group-size threshold would give.

    python tools/levels_compare.py 4 gpurun_out/f_lv4_all.json gpurun_out/f_lv4_none.json
"""
import json
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for  # noqa: E402

cfg = int(sys.argv[1])
A = json.load(open(sys.argv[2]))["launches"]
B = json.load(open(sys.argv[3]))["launches"]
p = config_problem(cfg, 1)
plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
g = plan.groups


def per_group(L):
    d = defaultdict(float)
    for x in L:
        d[(x["group"], x["kind"])] += x["ms"]
    return d


a, b = per_group(A), per_group(B)
kinds = sorted({k for _, k in a} | {k for _, k in b})
print("kind         A(ms)     B(ms)")
for k in kinds:
    print(f"{k:10s} {sum(v for (gg, kk), v in a.items() if kk == k):9.2f} {sum(v for (gg, kk), v in b.items() if kk == k):9.2f}")
print("total      ", round(sum(a.values()), 2), round(sum(b.values()), 2))
for kind, key in (("trail", "max_n"), ("rgemm", "max_s"), ("schur", "max_s"), ("tgemm", "max_s")):
    rows = []
    for thr in (0, 64, 128, 192, 256, 384, 512, 768, 1024, 1536, 100000):
        t = 0.0
        for (gi, kk), v in b.items():
            if kk != kind:
                continue
            use_a = int(g[key][gi]) >= thr
            t += a.get((gi, kk), v) if use_a else v
        rows.append((thr, round(t, 2)))
    print(kind, "threshold on", key, "-> ms:", rows)
