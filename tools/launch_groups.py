"""Annotate an ncu launch list (profile_step.py, last solve) with the plan's launch table.

    python tools/launch_groups.py launches.csv [--config 1]
Prints time per (pass, level, group) and per launch kind inside the heaviest groups.
"""
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from launch_summary import load  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import Plan  # noqa: E402

cfg = int(sys.argv[sys.argv.index("--config") + 1]) if "--config" in sys.argv else 1
p = config_problem(cfg, 1)
plan = Plan(p.nx, p.ny, p.indptr, p.indices)
sp = plan.specs(int(sys.argv[sys.argv.index("--energies") + 1]) if "--energies" in sys.argv else 16)
L = len(sp["kind"])
data = load(sys.argv[1])
data = data[len(data) - L:]
g = plan.groups
per_group = collections.defaultdict(float)
per_gk = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0.0]))
for i, (name, us, grid) in enumerate(data):
    gi = int(sp["group"][i])
    per_group[gi] += us
    kk = Plan.KIND_NAMES[sp["kind"][i]]
    per_gk[gi][kk][0] += 1
    per_gk[gi][kk][1] += us
tot = sum(per_group.values())
print(f"total {tot:.0f} us over {L} launches")
for gi, us in sorted(per_group.items(), key=lambda kv: -kv[1])[:14]:
    desc = ", ".join(f"{k}:{v[0]}x{v[1] / max(v[0], 1):.0f}" for k, v in sorted(per_gk[gi].items(), key=lambda kv: -kv[1][1]))
    print(f"g{gi:3d} pass{g['pass'][gi]} L{g['level'][gi]:2d} path{g['path'][gi]} n={g['count'][gi]:5d} "
          f"s<={g['max_s'][gi]:4d} b<={g['max_b'][gi]:4d} {us:8.0f} us ({100 * us / tot:4.1f}%)  {desc}")
