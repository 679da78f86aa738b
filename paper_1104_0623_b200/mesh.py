"""Mesh and the nested-dissection cluster tree (drop-in for find_selinv/mesh.py).

The tree and all node sets are built natively by the plan builder
(csrc/plan.cpp, restating mesh.py:176-290); this module exposes them with the
reference's names and fields for callers and tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


@dataclass(frozen=True)
class Mesh:
    """A 2D Cartesian grid with row-major node numbering (mesh.py:33-82)."""

    nx: int
    ny: int

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ValueError(f"mesh dimensions must be positive, got {self.nx}x{self.ny}")

    @property
    def n(self) -> int:
        return self.nx * self.ny

    def node_id(self, x: int, y: int) -> int:
        if not (0 <= x < self.nx and 0 <= y < self.ny):
            raise ValueError(f"coordinates ({x},{y}) outside {self.nx}x{self.ny} mesh")
        return x + self.nx * y

    def node_xy(self, node: int) -> tuple[int, int]:
        if not (0 <= node < self.n):
            raise ValueError(f"node id {node} out of range")
        return node % self.nx, node // self.nx

    def neighbors(self, node: int) -> np.ndarray:
        x, y = self.node_xy(node)
        out = []
        if y > 0:
            out.append(node - self.nx)
        if x > 0:
            out.append(node - 1)
        if x < self.nx - 1:
            out.append(node + 1)
        if y < self.ny - 1:
            out.append(node + self.nx)
        return np.array(out, dtype=np.int64)

    def adjacency(self) -> sp.csr_matrix:
        ids = np.arange(self.n, dtype=np.int64).reshape(self.ny, self.nx)
        hl, hr = ids[:, :-1].ravel(), ids[:, 1:].ravel()
        vl, vh = ids[:-1, :].ravel(), ids[1:, :].ravel()
        rows = np.concatenate([hl, hr, vl, vh])
        cols = np.concatenate([hr, hl, vh, vl])
        return sp.coo_matrix((np.ones(rows.size, dtype=np.int8), (rows, cols)), shape=(self.n, self.n)).tocsr()


def build_mesh(nx: int, ny: int) -> Mesh:
    return Mesh(nx, ny)


@dataclass(eq=False)
class Cluster:
    """One cluster of the tree with its node sets (mesh.py:89-118)."""

    label: int
    x0: int
    y0: int
    width: int
    height: int
    level: int
    children: tuple = ()
    parent: "Cluster | None" = field(default=None, repr=False)
    nodes: np.ndarray = field(default=None, repr=False)
    boundary: np.ndarray | None = field(default=None, repr=False)
    inner: np.ndarray | None = field(default=None, repr=False)
    private_inner: np.ndarray | None = field(default=None, repr=False)

    @property
    def is_leaf(self) -> bool:
        return not self.children

    @property
    def size(self) -> int:
        return self.width * self.height


@dataclass
class ComplementCluster:
    label: int
    boundary: np.ndarray
    private_inner: np.ndarray


class ClusterTree:
    """Binary nested-dissection tree (mesh.py:136-167), node sets read from a native plan."""

    def __init__(self, mesh: Mesh, root: Cluster, leaf_max: int):
        self.mesh = mesh
        self.root = root
        self.leaf_max = leaf_max
        self.by_label: dict[int, Cluster] = {}
        self.leaves: list[Cluster] = []
        for c in self.clusters():
            self.by_label[c.label] = c
            if c.is_leaf:
                self.leaves.append(c)
        self.annotated = root.boundary is not None

    def clusters(self):
        stack = [self.root]
        while stack:
            c = stack.pop()
            yield c
            stack.extend(reversed(c.children))

    def bottom_up(self):
        return sorted(self.by_label.values(), key=lambda c: (-c.level, c.label))

    def sibling(self, cluster: Cluster) -> Cluster:
        from .errors import TreeStateError

        if cluster.parent is None:
            raise TreeStateError("root has no sibling")
        a, b = cluster.parent.children
        return b if a is cluster else a


def _rect_geometry(nx, ny, leaf_max):
    """mesh.py:176-206 split rule (geometry only; sets come from the plan)."""
    out = []

    def make(label, x0, y0, w, h, level, parent):
        c = Cluster(label, x0, y0, w, h, level, parent=parent)
        ys = np.arange(y0, y0 + h, dtype=np.int64) * nx
        xs = np.arange(x0, x0 + w, dtype=np.int64)
        c.nodes = (ys[:, None] + xs[None, :]).ravel()
        out.append(c)
        if w <= leaf_max and h <= leaf_max:
            return c
        if w >= h:
            wl = (w + 1) // 2
            c.children = (make(2 * label, x0, y0, wl, h, level + 1, c), make(2 * label + 1, x0 + wl, y0, w - wl, h, level + 1, c))
        else:
            hl = (h + 1) // 2
            c.children = (make(2 * label, x0, y0, w, hl, level + 1, c), make(2 * label + 1, x0, y0 + hl, w, h - hl, level + 1, c))
        return c

    return make(1, 0, 0, nx, ny, 0, None)


def build_cluster_tree(mesh: Mesh, leaf_max: int) -> ClusterTree:
    """Unannotated tree with the reference's split rule and heap labels."""
    if leaf_max < 1:
        raise ValueError(f"leaf_max must be >= 1, got {leaf_max}")
    return ClusterTree(mesh, _rect_geometry(mesh.nx, mesh.ny, leaf_max), leaf_max)


def annotated_tree(plan) -> tuple[ClusterTree, dict[int, ComplementCluster]]:
    """Tree + complement sets filled from a native plan (mesh.py:255-290 semantics)."""
    tree = build_cluster_tree(Mesh(plan.nx, plan.ny), plan.leaf_max)
    comps = {}
    for c in tree.by_label.values():
        c.boundary = plan.cluster_set(c.label, 1)
        c.private_inner = plan.cluster_set(c.label, 2)
        c.inner = np.setdiff1d(c.nodes, c.boundary, assume_unique=True)
        comps[-c.label] = ComplementCluster(-c.label, plan.cluster_set(c.label, 3), plan.cluster_set(c.label, 4))
    tree.annotated = True
    return tree, comps
