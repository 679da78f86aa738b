"""Host handle of the native, energy-independent FIND plan.

The plan replaces the reference's per-solve set-up (build_cluster_tree +
annotate_boundaries + complement_boundary_sets, mesh.py:176-290, and the
merge bookkeeping of solver.py:97-132, 234-243) with one native build per
sparsity pattern, cached and reused across energy points and calls.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import threading
import time
from fractions import Fraction

import numpy as np

from . import _native
from .errors import NativeLibraryError, SingularPivotError
from .ledger import FlopLedger, plan_ledger

_INFO_KEYS = ("n", "nnz", "n_clusters", "n_elims", "n_levels_up", "n_levels_down", "up_arena_elems",
              "down_arena_elems", "ws_elems", "max_n", "max_s", "max_b", "n_groups", "sparse_entries", "depth",
              "n_leaves")


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class Plan:
    """Native plan for one (mesh, CSR pattern, leaf_max)."""

    def __init__(self, nx: int, ny: int, indptr: np.ndarray, indices: np.ndarray, leaf_max: int = 2):
        L = _native.lib()
        self.nx, self.ny, self.leaf_max = int(nx), int(ny), int(leaf_max)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int64)
        st = _native.FindStatus()
        h = C.c_void_p()
        t0 = time.perf_counter()
        rc = L.find_plan_create(self.nx, self.ny, _i64p(self.indptr), _i64p(self.indices), self.indices.size,
                                self.leaf_max, C.byref(h), C.byref(st))
        self.build_seconds = time.perf_counter() - t0
        if rc != _native.FIND_OK:
            raise ValueError(st.text)
        self._h = h
        info = np.zeros(16, np.int64)
        L.find_plan_info(h, _i64p(info))
        self.info = dict(zip(_INFO_KEYS, (int(x) for x in info)))
        ne = self.info["n_elims"]
        self.kind = np.zeros(ne, np.int32)
        self.s = np.zeros(ne, np.int32)
        self.b = np.zeros(ne, np.int32)
        self.label = np.zeros(ne, np.int64)
        L.find_plan_elims(h, _i32p(self.kind), _i32p(self.s), _i32p(self.b), _i64p(self.label))
        ng = self.info["n_groups"]
        g = {k: np.zeros(ng, np.int32) for k in ("pass", "level", "path", "max_n", "max_s", "max_b")}
        cnt = np.zeros(ng, np.int64)
        L.find_plan_groups(h, _i32p(g["pass"]), _i32p(g["level"]), _i32p(g["path"]), _i64p(cnt), _i32p(g["max_n"]),
                           _i32p(g["max_s"]), _i32p(g["max_b"]))
        g["count"] = cnt
        self.groups = g
        self.first_down_group = int(np.argmax(g["pass"] > 0)) if (g["pass"] > 0).any() else ng
        self._exc = {}
        self._ws = None
        self._lock = threading.Lock()
        self.cache: dict = {}  # per-pattern host-side caches (validation, maps, ledgers)
        self._pin_in = None
        self._pin_out = None
        self._dev_bufs: dict = {}  # persistent device buffers of solve_values (graph-stable pointers)
        self._graphs: dict = {}    # captured CUDA graphs of the level schedule, per (groups, shapes, pointers)
        self._graph_seen: dict = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _native.lib().find_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def n(self) -> int:
        return self.nx * self.ny

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    @property
    def handle(self):
        return self._h

    def cluster_set(self, label: int, which: int) -> np.ndarray:
        L = _native.lib()
        size = L.find_plan_cluster_set(self._h, int(label), int(which), None, 0)
        if size < 0:
            raise KeyError(label)
        out = np.zeros(max(size, 1), np.int64)
        L.find_plan_cluster_set(self._h, int(label), int(which), _i64p(out), size)
        return out[:size]

    def exception_slots(self, pass_: int) -> np.ndarray:
        if pass_ not in self._exc:
            L = _native.lib()
            k = L.find_plan_exception_slots(self._h, pass_, None, 0)
            out = np.zeros(max(k, 1), np.int64)
            L.find_plan_exception_slots(self._h, pass_, _i64p(out), k)
            self._exc[pass_] = out[:k]
        return self._exc[pass_]

    def ledger(self, kernel="naive", compute_gless=True, sigma_hermitian=False, sigma_mode="auto") -> FlopLedger:
        return plan_ledger(self.kind, self.s, self.b, kernel, compute_gless, sigma_hermitian, sigma_mode)

    def native_work(self, kernel_id: int = 0, compute_gless: bool = True) -> Fraction:
        """Exact per-energy W from the native ledger (naive / block kernels)."""
        num = np.zeros(_native.LEDGER_KEYS, np.int64)
        den = np.zeros(1, np.int64)
        rc = _native.lib().find_plan_ledger(self._h, kernel_id, int(compute_gless), _i64p(num), _i64p(den))
        if rc:
            raise ValueError("find_plan_ledger failed")
        return sum((Fraction(int(v), int(den[0])) for v in num), Fraction(0))

    def workspace_bytes(self, n_energies: int, compute_gless: bool = True) -> int:
        return int(_native.lib().find_solve_workspace_bytes(self._h, n_energies, int(compute_gless)))

    def launch_count(self, n_energies: int = 1) -> int:
        return int(_native.lib().find_solve_launch_count(self._h, int(n_energies)))

    KIND_NAMES = ("warp", "gatherA", "panel", "trsm", "trail", "xsolve", "finish", "gatherS", "tgemm", "rgemm", "final",
                  "schur", "lu_fused", "mid", "offdiag", "panel_inv")

    def offdiag_pairs(self) -> np.ndarray:
        """Directed adjacent pairs [n_pairs, 2] (u, v), u != v, ascending: the index space of the
        off-diagonal outputs (a.adjacency(), operators.py:84-93; solver.py:454-484)."""
        pr = self.cache.get("offdiag_pairs")
        if pr is None:
            L = _native.lib()
            k = L.find_plan_offdiag_pairs(self._h, None, None, 0)
            if k < 0:
                raise NativeLibraryError("find_plan_offdiag_pairs failed")
            u = np.zeros(max(k, 1), np.int64)
            v = np.zeros(max(k, 1), np.int64)
            L.find_plan_offdiag_pairs(self._h, _i64p(u), _i64p(v), k)
            pr = np.stack([u[:k], v[:k]], axis=1)
            self.cache["offdiag_pairs"] = pr
        return pr

    def group_phases(self) -> np.ndarray:
        """Phase of every launch group (groups of a phase are independent; phases run in order)."""
        ph = np.zeros(len(self.groups["count"]), np.int32)
        _native.lib().find_plan_group_phases(self._h, _i32p(ph))
        return ph

    def specs(self, n_energies: int = 1) -> dict:
        """Kernel-launch table of a solve over n_energies points, in issue order."""
        k = self.launch_count(n_energies)
        out = {x: np.zeros(k, np.int32) for x in ("kind", "step", "group")}
        tasks = np.zeros(k, np.int64)
        _native.lib().find_plan_specs(self._h, int(n_energies), _i32p(out["kind"]), _i32p(out["step"]),
                                      _i32p(out["group"]), _i64p(tasks))
        out["tasks"] = tasks
        return out

    # ---- reused pinned host buffers for the H2D / D2H copies of solve_values ----
    def host_values(self, n_energies: int) -> np.ndarray:
        """A pinned [n_energies, nnz] complex128 host buffer (numpy view), reused across calls."""
        import torch

        if self._pin_in is None or self._pin_in.shape[0] < n_energies:
            t = torch.empty((n_energies, self.nnz), dtype=torch.complex128)
            self._pin_in = t.pin_memory() if torch.cuda.is_available() else t
        return self._pin_in[:n_energies].numpy()

    def is_pinned_view(self, arr: np.ndarray) -> bool:
        if self._pin_in is None or not self._pin_in.is_pinned():
            return False
        return arr.__array_interface__["data"][0] == self._pin_in.data_ptr()

    def pinned_tensor(self, arr: np.ndarray):
        return self._pin_in[: arr.shape[0]]

    def host_outputs(self, n_energies: int, compute_gless: bool):
        import torch

        if self._pin_out is None or self._pin_out[0].shape[0] < n_energies:
            self._pin_out = tuple(torch.empty((n_energies, self.n), dtype=torch.complex128).pin_memory()
                                  for _ in range(2))
        return self._pin_out[0][:n_energies], self._pin_out[1][:n_energies]

    # ---- device execution (torch tensors for memory/streams only) ----
    def workspace(self, n_energies: int, compute_gless: bool, device):
        import torch

        need = self.workspace_bytes(n_energies, compute_gless)
        with self._lock:
            if self._ws is None or self._ws.numel() < need or self._ws.device != device:
                self._ws = None
                self._graphs.clear()  # captured graphs point into the old workspace
                self._graph_seen.clear()
                try:
                    self._ws = torch.empty(need, dtype=torch.uint8, device=device)
                except torch.OutOfMemoryError:
                    release_workspaces(keep=self)  # workspaces cached by other plans
                    self._ws = torch.empty(need, dtype=torch.uint8, device=device)
            return self._ws

    def solve_stream(self, device):
        """A non-default CUDA stream owned by the plan (graph capture needs one)."""
        import torch

        st = self.cache.get(("stream", str(device)))
        if st is None:
            st = torch.cuda.Stream(device)
            self.cache[("stream", str(device))] = st
        return st

    def device_buffer(self, name: str, shape: tuple, device):
        """A persistent complex128 device tensor owned by the plan (stable address for graph replay)."""
        import torch

        key = (name, tuple(shape), str(device))
        t = self._dev_bufs.get(key)
        if t is None:
            t = torch.empty(shape, dtype=torch.complex128, device=device)
            self._dev_bufs[key] = t
        return t

    def replay_or_run(self, key, stream, fn):
        """Run fn() (stream-ordered work on `stream` into fixed buffers) eagerly the first time a
        key is seen; the second time capture it into a CUDA graph; afterwards replay the graph:
        one launch instead of ~2000 host-side kernel launches per solve.  FIND_B200_GRAPH=0 off."""
        import os

        import torch

        if os.environ.get("FIND_B200_GRAPH", "1") == "0":
            return fn()
        g = self._graphs.get(key)
        if g is not None:
            g.replay()
            return None
        n = self._graph_seen.get(key, 0) + 1
        self._graph_seen[key] = n
        if n < 2:
            return fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        self._graphs[key] = g
        g.replay()
        return None

    def run(self, a_dev, s_dev, gr_dev, gl_dev, compute_gless=True, pivot_rtol=1e-12, s_broadcast=True, ws=None,
            stream=None, groups=(0, -1), check=True, sigma_sym=0, off_gr=None, off_gl=None):
        """Enqueue the solve on `stream` for a_dev [nE, nnz] (torch complex128, CUDA).

        sigma_sym: +1 if Sigma^< is exactly Hermitian, -1 if exactly skew-Hermitian
        (then every R block is too and only its lower triangle is computed).
        off_gr / off_gl: optional CUDA complex128 [nE, n_pairs] outputs of G^r / G^< on
        offdiag_pairs() (find_solve_offdiag)."""
        import torch

        L = _native.lib()
        if not a_dev.is_cuda or a_dev.dtype != torch.complex128 or a_dev.dim() != 2 or a_dev.shape[1] != self.nnz:
            raise ValueError("a_dev must be a CUDA complex128 tensor of shape [n_energies, nnz]")
        n_e = int(a_dev.shape[0])
        if ws is None:
            ws = self.workspace(n_e, compute_gless, a_dev.device)
        if stream is None:
            stream = torch.cuda.current_stream(a_dev.device)
        st = _native.FindStatus()
        cg = 0 if not compute_gless else {1: 2, -1: 3}.get(int(sigma_sym), 1)
        head = (self._h, C.c_void_p(a_dev.data_ptr()), C.c_void_p(s_dev.data_ptr() if s_dev is not None else 0),
                int(s_broadcast), n_e, cg, float(pivot_rtol), C.c_void_p(gr_dev.data_ptr()),
                C.c_void_p(gl_dev.data_ptr() if gl_dev is not None else 0))
        tail = (C.c_void_p(ws.data_ptr()), ws.numel(), int(groups[0]), int(groups[1]), C.c_void_p(stream.cuda_stream),
                C.byref(st))
        if off_gr is None:
            rc = L.find_solve_groups(*head, *tail)
        else:
            rc = L.find_solve_offdiag_groups(*head, C.c_void_p(off_gr.data_ptr()),
                                             C.c_void_p(off_gl.data_ptr() if off_gl is not None else 0), *tail)
        if rc != _native.FIND_OK:
            if rc == _native.FIND_EINVAL:
                raise ValueError(st.text)
            raise NativeLibraryError(f"find_solve failed ({rc}): {st.text}")
        return ws

    def check_status(self, ws, n_energies, stream=None):
        import torch

        if stream is None:
            stream = torch.cuda.current_stream(ws.device)
        st = _native.FindStatus()
        rc = _native.lib().find_solve_status(self._h, C.c_void_p(ws.data_ptr()), n_energies,
                                             C.c_void_p(stream.cuda_stream), C.byref(st))
        if rc == _native.FIND_ESINGULAR:
            raise SingularPivotError(st.text, node=(int(st.node_id) if st.node_id >= 0 else None),
                                     cluster=int(st.cluster_label), energy=int(st.energy_idx))
        if rc != _native.FIND_OK:
            raise NativeLibraryError(f"find_solve_status failed ({rc}): {st.text}")


_CACHE: dict = {}
_CACHE_LOCK = threading.Lock()


def release_workspaces(keep: "Plan | None" = None) -> None:
    """Drop the device workspaces cached by every plan except ``keep`` and return the memory."""
    import torch

    with _CACHE_LOCK:
        plans = list(_CACHE.values())
    for p in plans:
        if p is not keep:
            p._ws = None
            p._graphs.clear()
            p._graph_seen.clear()
            p._dev_bufs.clear()
    if torch.cuda.is_available():
        torch.cuda.empty_cache()


_LAST: list = []  # (nx, ny, leaf_max, indptr, indices, plan) of the last lookup: memcmp fast path


_libc = C.CDLL(None)
_libc.memcmp.restype = C.c_int
_libc.memcmp.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]


def same_array(a: np.ndarray, b: np.ndarray) -> bool:
    """a == b element for element; one memcmp (GIL released) when dtype and layout match."""
    if a is b:
        return True
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype == b.dtype and a.flags.c_contiguous and b.flags.c_contiguous and a.dtype.kind in "iub":
        return a.nbytes == 0 or _libc.memcmp(a.ctypes.data, b.ctypes.data, a.nbytes) == 0
    return bool(np.array_equal(a, b))


def plan_for(nx: int, ny: int, indptr: np.ndarray, indices: np.ndarray, leaf_max: int = 2) -> tuple[Plan, float]:
    """Cached plan for a pattern; returns (plan, seconds spent building it now)."""
    if _LAST:
        lx, ly, ll, lp, li, lplan = _LAST[0]
        if (lx, ly, ll) == (int(nx), int(ny), int(leaf_max)) and lp.size == np.size(indptr) and li.size == np.size(
                indices) and same_array(lp, indptr) and same_array(li, indices):
            return lplan, 0.0
    p, t = _plan_for_hashed(nx, ny, indptr, indices, leaf_max)
    _LAST[:] = [(int(nx), int(ny), int(leaf_max), p.indptr, p.indices, p)]
    return p, t


def _plan_for_hashed(nx: int, ny: int, indptr: np.ndarray, indices: np.ndarray, leaf_max: int = 2):
    h = hashlib.sha1()
    h.update(np.ascontiguousarray(indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(indices, dtype=np.int64).tobytes())
    key = (int(nx), int(ny), int(leaf_max), h.hexdigest())
    with _CACHE_LOCK:
        p = _CACHE.get(key)
        if p is not None:
            return p, 0.0
    p = Plan(nx, ny, indptr, indices, leaf_max)
    with _CACHE_LOCK:
        if len(_CACHE) > 16:
            _CACHE.clear()
        _CACHE[key] = p
    return p, p.build_seconds
