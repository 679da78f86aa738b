import os, sys
sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo')
import numpy as np
from test_gpu import shim, dense_input, ref_update, rel
import torch
for nb in ("32", "16", "8"):
    os.environ["FIND_B200_NB"] = nb
    for s, b in [(20, 15), (40, 30), (100, 90), (250, 60), (257, 60), (300, 40), (520, 30)]:
        ass, asb, abs_, abb = dense_input(s, b, seed=s * 131 + b)
        rng = np.random.default_rng(s + 7 * b); n = s + b
        sm = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        rc, st, u, r, l = shim(ass, asb, abs_, abb, sm[:s,:s], sm[:s,s:], sm[s:,:s], sm[s:,s:], path=1)
        ue, re_, le = ref_update(ass, asb, abs_, abb, sm[:s,:s], sm[:s,s:], sm[s:,:s], sm[s:,s:])
        print(nb, s, b, rc, f"u {rel(u, ue):.1e} r {rel(r, re_):.1e} l {rel(l, le):.1e}", flush=True)
