"""CSR graphs: the reference's ``hyperanf::Graph`` surface (graph.hpp:23-229).

A :class:`Graph` holds numpy arrays ``offsets`` (u64, n+1) and ``arcs`` (u32);
construction, the reference fixtures, the BASELINE synthetic configs and the
HBG1 cache go through libhanf.so's host code.
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, c_uint32, c_uint64, c_void_p

import numpy as np

from . import _lib
from ._lib import check, lib


class _GraphHandle:
    """Owns a hanf_graph; freed when no array views it any more."""

    def __init__(self, handle: c_void_p):
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                lib().hanf_graph_free(self.handle)
        except Exception:
            pass


class _CsrBuffer:
    """Buffer exporter (PEP 688) for one array of a library-built graph; the
    arrays created from it keep the owning _GraphHandle alive."""

    def __init__(self, owner: _GraphHandle, ptr, count: int, ctype):
        self.owner = owner
        self.carr = (ctype * count).from_address(ctypes.cast(ptr, ctypes.c_void_p).value)

    def __buffer__(self, flags):
        return memoryview(self.carr)

    def __release_buffer__(self, view):
        pass


class Graph:
    """Immutable directed graph in CSR layout (graph.hpp:23-69)."""

    __slots__ = ("_n", "_offsets", "_arcs", "_pinned")

    def __init__(self, n: int = 0, offsets=None, arcs=None):
        self._pinned = []
        self._n = int(n)
        self._offsets = (np.zeros(1, dtype=np.uint64) if offsets is None
                         else np.ascontiguousarray(offsets, dtype=np.uint64))
        self._arcs = (np.zeros(0, dtype=np.uint32) if arcs is None
                      else np.ascontiguousarray(arcs, dtype=np.uint32))
        if self._offsets.shape != (self._n + 1,):
            raise ValueError("offsets must have n + 1 entries")
        if int(self._offsets[-1]) != self._arcs.size:
            raise ValueError("offsets[n] must equal the arc count")

    # -- construction -----------------------------------------------------
    @staticmethod
    def _adopt(handle: c_void_p) -> "Graph":
        """Wraps a library-built graph without copying it: the numpy arrays
        view the C++ CSR, which is freed when the last view is gone (a
        config-5 graph is 19 GB)."""
        view = _lib.GraphView()
        try:
            check(lib().hanf_graph_view_of(handle, ctypes.byref(view)))
        except Exception:
            lib().hanf_graph_free(handle)
            raise
        owner = _GraphHandle(handle)
        n = int(view.n)
        offsets = np.frombuffer(_CsrBuffer(owner, view.offsets, n + 1, ctypes.c_uint64),
                                dtype=np.uint64)
        arcs = (np.frombuffer(_CsrBuffer(owner, view.arcs, int(view.num_arcs), ctypes.c_uint32),
                              dtype=np.uint32)
                if view.num_arcs else np.zeros(0, dtype=np.uint32))
        return Graph(n, offsets, arcs)

    @staticmethod
    def from_edges(n: int, edges, device: int = None) -> "Graph":
        """graph.hpp:29-44: sorts each successor list and collapses duplicates.
        device=k builds the same CSR with device radix sorts on GPU k."""
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if e.size and (e.min() < 0 or e.max() >= n):
            raise ValueError("arc endpoint out of range")
        src = np.ascontiguousarray(e[:, 0], dtype=np.uint32)
        dst = np.ascontiguousarray(e[:, 1], dtype=np.uint32)
        h = c_void_p()
        args = (n, src.ctypes.data_as(POINTER(c_uint32)), dst.ctypes.data_as(POINTER(c_uint32)),
                src.size, ctypes.byref(h))
        if device is None:
            check(lib().hanf_graph_from_edges(*args))
        else:
            check(lib().hanf_graph_from_edges_gpu(device, *args))
        return Graph._adopt(h)

    # -- page-locking for uploads (new; hanf_pin_host) -------------------------
    def pin(self) -> "Graph":
        """Page-locks the CSR arrays in place so engines upload them by DMA
        at full link rate; undone by unpin() or when the graph is freed."""
        for arr in (self._offsets, self._arcs):
            if arr.nbytes and not any(p == arr.ctypes.data for p in self._pinned):
                check(lib().hanf_pin_host(c_void_p(arr.ctypes.data), arr.nbytes))
                self._pinned.append(arr.ctypes.data)
        return self

    def unpin(self) -> None:
        while self._pinned:
            check(lib().hanf_unpin_host(c_void_p(self._pinned.pop())))

    def __del__(self):
        try:
            if getattr(self, "_pinned", None):
                self.unpin()
        except Exception:
            pass

    # -- accessors (graph.hpp:46-57) ----------------------------------------
    def num_nodes(self) -> int:
        return self._n

    def num_arcs(self) -> int:
        return int(self._arcs.size)

    def successors(self, v: int) -> np.ndarray:
        return self._arcs[int(self._offsets[v]):int(self._offsets[v + 1])]

    def out_degree(self, v: int) -> int:
        return int(self._offsets[v + 1] - self._offsets[v])

    def offsets(self) -> np.ndarray:
        return self._offsets

    def arcs(self) -> np.ndarray:
        return self._arcs

    def __eq__(self, other) -> bool:
        return (isinstance(other, Graph) and self._n == other._n
                and np.array_equal(self._offsets, other._offsets)
                and np.array_equal(self._arcs, other._arcs))

    def view(self) -> _lib.GraphView:
        """hanf_graph_view over this graph's arrays (borrowed, no copy)."""
        v = _lib.GraphView()
        v.n = self._n
        v.num_arcs = self._arcs.size
        v.offsets = self._offsets.ctypes.data_as(POINTER(c_uint64))
        v.arcs = self._arcs.ctypes.data_as(POINTER(c_uint32))
        return v

    def _handle(self) -> c_void_p:
        h = c_void_p()
        src = np.repeat(np.arange(self._n, dtype=np.uint32),
                        np.diff(self._offsets).astype(np.int64))
        check(lib().hanf_graph_from_edges(
            self._n, src.ctypes.data_as(POINTER(c_uint32)),
            self._arcs.ctypes.data_as(POINTER(c_uint32)), self._arcs.size, ctypes.byref(h)))
        return h


def transpose(g: Graph) -> Graph:
    """graph.hpp:72-84: arc y->x for every arc x->y."""
    h = g._handle()
    t = c_void_p()
    try:
        check(lib().hanf_graph_transpose(h, ctypes.byref(t)))
    finally:
        lib().hanf_graph_free(h)
    return Graph._adopt(t)


def gen_uniform_random(n: int, d: float, seed: int) -> Graph:
    """graph.hpp:262-285 (same bits as the reference)."""
    h = c_void_p()
    check(lib().hanf_gen_uniform_random(n, float(d), seed, ctypes.byref(h)))
    return Graph._adopt(h)


def gen_clique_path(k: int, l: int) -> Graph:
    """graph.hpp:238-258 (same bits as the reference)."""
    h = c_void_p()
    check(lib().hanf_gen_clique_path(k, l, ctypes.byref(h)))
    return Graph._adopt(h)


def gen_erdos_renyi(n: int, mean_degree: float, seed: int) -> Graph:
    """BASELINE config 1: directed G(n, p), p = mean_degree/(n-1), no self-loops."""
    h = c_void_p()
    check(lib().hanf_gen_erdos_renyi(n, float(mean_degree), seed, ctypes.byref(h)))
    return Graph._adopt(h)


def gen_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
             c: float = 0.19, seed: int = 1, permute_seed: int = 7, device: int = None) -> Graph:
    """BASELINE configs 2/5: R-MAT, self-loops and duplicates removed, ids
    permuted.  device=k generates the same graph on GPU k (hanf_gen_rmat_gpu)."""
    h = c_void_p()
    if device is None:
        check(lib().hanf_gen_rmat(scale, edge_factor, a, b, c, seed, permute_seed,
                                  ctypes.byref(h)))
    else:
        check(lib().hanf_gen_rmat_gpu(device, scale, edge_factor, a, b, c, seed, permute_seed,
                                      ctypes.byref(h)))
    return Graph._adopt(h)


def gen_copying(n: int, exponent: float = 2.1, mean_degree: float = 20.0,
                max_degree: int = 5000, copy_prob: float = 0.6, window: int = 1 << 12,
                seed: int = 3) -> Graph:
    """BASELINE config 3: web-like copying model (Workloads)."""
    h = c_void_p()
    check(lib().hanf_gen_copying(n, exponent, mean_degree, max_degree, copy_prob, window,
                                 seed, ctypes.byref(h)))
    return Graph._adopt(h)


def gen_barabasi_albert(n: int, m: int = 10, seed: int = 4, permute_seed: int = 11) -> Graph:
    """BASELINE config 4: symmetric Barabasi-Albert, ids permuted."""
    h = c_void_p()
    check(lib().hanf_gen_barabasi_albert(n, m, seed, permute_seed, ctypes.byref(h)))
    return Graph._adopt(h)


def save_csr(g: Graph, path: str) -> None:
    """HBG1 cache writer (graph.hpp:178-187)."""
    h = g._handle()
    try:
        check(lib().hanf_graph_save_csr(h, path.encode()))
    finally:
        lib().hanf_graph_free(h)


def load_csr(path: str) -> Graph:
    """HBG1 cache reader (graph.hpp:196-218)."""
    h = c_void_p()
    check(lib().hanf_graph_load_csr(path.encode(), ctypes.byref(h)))
    return Graph._adopt(h)
