"""Executed-work model of one solve, per launch kind (for the roofline in bench.py).

Counts the complex multiply-adds each kernel kind actually performs, from the
plan's (s, b) per elimination and the group panel width; ``x 8`` gives real
FP64 flops.  This is the kernels' own arithmetic (e.g. the Schur launch does
s*b^2 = the sb^2 term of the reference's naive_dense count, kernels.py:90),
distinct from the paper's ledger W that ``fp64_tflops`` is quoted on.  The structural-zero
skips (ElimDesc::zsplit: Schur K from |S_l|, trailing / L21 tiles of B_r rows) are not
subtracted: they remove about 4 % of the Schur MACs on cfg1 (find_plan_elim_splits).
"""

from __future__ import annotations

import numpy as np

KINDS = ("warp", "gatherA", "panel", "trsm", "trail", "xsolve", "finish", "gatherS", "tgemm", "rgemm", "final",
         "schur", "lu_fused", "mid", "offdiag", "panel_inv")
TENSOR_KINDS = ("trsm", "trail", "xsolve", "tgemm", "rgemm", "schur")


def pick_nb(max_s: int) -> int:
    """Mirror of pick_nb_host (csrc/plan.h)."""
    if max_s <= 8 * 384:  # register / shared-memory / cluster panels (csrc/plan.h pick_nb_host)
        return 32
    for nb, w in ((16, 17), (8, 9), (4, 5)):
        if max_s * w * 16 <= 220 * 1024:
            return nb
    return 0


def _dense_elim(s, b, sym):
    n = s + b
    lu = sum((n - k - 1) ** 2 for k in range(s))
    x = b * s * (s - 1) // 2
    t = b * s * s
    r = 2 * s * (b * (b + 1) // 2 if sym else b * b)
    return lu + x + t + r


def executed_cmacs(plan, sigma_sym: int = 0) -> dict:
    """{(group, kind): complex MACs} for one energy point."""
    g = plan.groups
    start = np.concatenate([[0], np.cumsum(g["count"])])
    out = {}
    for gi in range(len(g["count"])):
        s_arr = plan.s[start[gi]:start[gi + 1]].astype(np.int64)
        b_arr = plan.b[start[gi]:start[gi + 1]].astype(np.int64)
        path = int(g["path"][gi])
        sym = sigma_sym != 0 and int(g["pass"][gi]) == 0
        if path in (0, 2):
            out[(gi, "warp" if path == 0 else "mid")] = float(sum(_dense_elim(int(s), int(b), sym)
                                                                 for s, b in zip(s_arr, b_arr)))
            continue
        nb = pick_nb(int(g["max_s"][gi]))
        acc = {k: 0.0 for k in ("panel", "trsm", "trail", "xsolve", "schur", "tgemm", "rgemm")}
        for s, b in zip(s_arr.tolist(), b_arr.tolist()):
            n = s + b
            for j0 in range(0, s, nb):
                jb = min(nb, s - j0)
                j1 = j0 + jb
                r = s - j0
                acc["panel"] += sum(max(r - jj - 1, 0) for jj in range(jb)) * (nb - 1)
                acc["trsm"] += jb * jb * (n - j1) + b * jb * jb
                acc["trail"] += ((n - j1) ** 2 - b * b) * jb
                acc["xsolve"] += b * jb * (s - j1) + b * jb * jb  # Z, then Z L_jj^-1 (DMMA)
            acc["schur"] += b * b * s
            acc["tgemm"] += b * s * s
            acc["rgemm"] += 2 * s * (b * (b + 1) // 2 if sym else b * b)
        for k, v in acc.items():
            out[(gi, k)] = v
    return out
