"""Data formats on either side of the solve (host side, no device work).

Matrix Market in / out (operators.py:222-244) and the CSV exports of a result
(solver.py:709-734), byte-compatible with the reference: values printed with
``format(x, ".17g")``, rows in node order / ascending (i, j).
"""

from __future__ import annotations

import numpy as np
import scipy.io
import scipy.sparse as sp

from .operators import SparseOperator


def write_matrix_market(path, op: SparseOperator, mesh=None) -> None:
    """operators.py:222-230: coordinate complex general; ``%%mesh nx ny`` records the grid."""
    comment = f"%mesh {mesh.nx} {mesh.ny}" if mesh is not None else ""
    scipy.io.mmwrite(path, op.matrix.tocoo(), comment=comment, field="complex", symmetry="general")


def read_matrix_market(path) -> tuple[SparseOperator, tuple[int, int] | None]:
    """operators.py:233-244: the operator and, if present, the ``%%mesh nx ny`` header."""
    dims = None
    with open(path, "r") as fh:
        for line in fh:
            if not line.startswith("%"):
                break
            if line.startswith("%%mesh"):
                parts = line.split()
                if len(parts) >= 3:
                    dims = (int(parts[1]), int(parts[2]))
    m = scipy.io.mmread(path)
    return SparseOperator(sp.csr_matrix(m)), dims


def _fmt(x: float) -> str:
    return format(x, ".17g")


def diag_to_csv(result, mesh, energy: int | None = None) -> str:
    """solver.py:713-726.  ``result`` is a SelectedInverse, or a SelectedInverseBatch
    with ``energy`` selecting the row."""
    gr = result.gr_diag if energy is None else result.gr_diag[energy]
    gl = result.gless_diag if energy is None or result.gless_diag is None else result.gless_diag[energy]
    n = mesh.n
    nodes = np.arange(n)
    xs, ys = (nodes % mesh.nx).tolist(), (nodes // mesh.nx).tolist()
    gre, gim = gr.real.tolist(), gr.imag.tolist()
    lines = ["node,x,y,re_gr,im_gr,re_gless,im_gless"]
    if gl is not None:
        lre, lim = gl.real.tolist(), gl.imag.tolist()
        lines += [f"{k},{xs[k]},{ys[k]},{_fmt(gre[k])},{_fmt(gim[k])},{_fmt(lre[k])},{_fmt(lim[k])}" for k in range(n)]
    else:
        lines += [f"{k},{xs[k]},{ys[k]},{_fmt(gre[k])},{_fmt(gim[k])},," for k in range(n)]
    return "\n".join(lines) + "\n"


def offdiag_to_csv(result, energy: int | None = None, gless: bool = False) -> str:
    """solver.py:729-734: ``i,j,re,im`` in ascending (i, j).  For a SelectedInverseBatch,
    ``energy`` selects the row; ``gless=True`` writes G^< instead of G^r."""
    lines = ["i,j,re,im"]
    if energy is None:
        d = result.offdiag_gless if gless else result.offdiag
        if d:
            for (i, j) in sorted(d):
                v = d[(i, j)]
                lines.append(f"{i},{j},{_fmt(v.real)},{_fmt(v.imag)}")
    else:
        vals = result.offdiag_gless if gless else result.offdiag_gr
        if vals is not None:
            pr = result.offdiag_pairs.tolist()
            v = vals[energy]
            re, im = v.real.tolist(), v.imag.tolist()
            lines += [f"{i},{j},{_fmt(re[k])},{_fmt(im[k])}" for k, (i, j) in enumerate(pr)]
    return "\n".join(lines) + "\n"
