"""Parity checkers for the B200 engine -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this package, and only as the checker or
the timed CPU baseline, never as the product path.

Two checkers, both built by oracle/Makefile:

* ``port``: liboracle.so, the plain-C restatement of the reference hot path
  (hanf_oracle.c, each function citing the reference file:line it follows);
* ``ref``:  _ref/libhanf_ref.so, the UNMODIFIED reference engine compiled
  from its own headers (ref_shim.cpp includes them by path; nothing is
  copied).  Available wherever the prebuilt .so travelled (the GPU box).

The port is pinned against ``ref`` and the golden fixtures in tests/golden.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libhanf_ref.so")


class _Params(ctypes.Structure):
    _fields_ = [("bucket_bits", ctypes.c_uint), ("registers", ctypes.c_uint),
                ("register_bits", ctypes.c_uint), ("alpha", c_double),
                ("seed", c_uint64), ("words", ctypes.c_uint)]


class _Graph(ctypes.Structure):
    _fields_ = [("n", c_uint64), ("arcs", c_uint64), ("offsets", POINTER(c_uint64)),
                ("succ", POINTER(c_uint32))]


class _Config(ctypes.Structure):
    _fields_ = [("bucket_bits", ctypes.c_uint), ("register_bits", ctypes.c_uint),
                ("seed", c_uint64), ("systolic_threshold", c_double),
                ("termination", c_int), ("eps_inc", c_double),
                ("max_iterations", c_uint64), ("track_modified", c_int),
                ("use_systolic", c_int)]


def _u64p(a):
    return a.ctypes.data_as(POINTER(c_uint64))


def _u32p(a):
    return a.ctypes.data_as(POINTER(c_uint32))


def _f64p(a):
    return a.ctypes.data_as(POINTER(c_double))


# --------------------------------------------------------------------------
# port: the C restatement
# --------------------------------------------------------------------------
class Port:
    def __init__(self, path: str = PORT_PATH):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle`")
        L = ctypes.CDLL(path)
        L.or_mix64.restype = c_uint64
        L.or_mix64.argtypes = [c_uint64]
        L.or_item_hash.restype = c_uint64
        L.or_item_hash.argtypes = [c_uint64, c_uint64]
        L.or_params_make.argtypes = [ctypes.c_uint, c_uint64, ctypes.c_uint, POINTER(_Params)]
        L.or_read_register.restype = ctypes.c_uint
        L.or_read_register.argtypes = [POINTER(c_uint64), POINTER(_Params), ctypes.c_uint]
        L.or_write_register.argtypes = [POINTER(c_uint64), POINTER(_Params), ctypes.c_uint,
                                        ctypes.c_uint]
        L.or_counter_add.argtypes = [POINTER(c_uint64), POINTER(_Params), c_uint64]
        L.or_counter_estimate.restype = c_double
        L.or_counter_estimate.argtypes = [POINTER(c_uint64), POINTER(_Params)]
        L.or_naive_union.argtypes = [POINTER(c_uint64), POINTER(c_uint64), POINTER(_Params)]
        L.or_packed_max_into.argtypes = [POINTER(_Params), POINTER(c_uint64), POINTER(c_uint64)]
        L.or_selftest_straddle.restype = c_uint64
        L.or_graph_from_edges.argtypes = [c_uint64, POINTER(c_uint32), POINTER(c_uint32),
                                          c_uint64, POINTER(_Graph)]
        L.or_graph_transpose.argtypes = [POINTER(_Graph), POINTER(_Graph)]
        L.or_gen_uniform_random.argtypes = [c_uint64, c_double, c_uint64, POINTER(_Graph)]
        L.or_gen_clique_path.argtypes = [c_uint64, c_uint64, POINTER(_Graph)]
        L.or_graph_free.argtypes = [POINTER(_Graph)]
        L.or_config_default.argtypes = [POINTER(_Config)]
        L.or_engine_create.restype = c_void_p
        L.or_engine_create.argtypes = [POINTER(c_uint64), POINTER(c_uint32), c_uint64,
                                       POINTER(_Config), POINTER(c_int)]
        L.or_engine_destroy.argtypes = [c_void_p]
        L.or_engine_sum_estimates.restype = c_double
        L.or_engine_sum_estimates.argtypes = [c_void_p]
        L.or_engine_step.argtypes = [c_void_p, POINTER(c_double), POINTER(c_uint64)]
        L.or_engine_counters.restype = POINTER(c_uint64)
        L.or_engine_counters.argtypes = [c_void_p]
        L.or_engine_words.restype = ctypes.c_uint
        L.or_engine_words.argtypes = [c_void_p]
        L.or_engine_iteration.restype = c_uint64
        L.or_engine_iteration.argtypes = [c_void_p]
        L.or_engine_systolic_active.argtypes = [c_void_p]
        L.or_engine_run.argtypes = [c_void_p, POINTER(c_double), POINTER(c_uint64), c_uint64,
                                    POINTER(c_uint64)]
        L.or_exact_nf.argtypes = [POINTER(c_uint64), POINTER(c_uint32), c_uint64,
                                  POINTER(c_uint64), c_uint64, POINTER(c_uint64)]
        L.or_clique_path_nf.restype = c_uint64
        L.or_clique_path_nf.argtypes = [c_uint64, c_uint64, c_uint64]
        L.or_counter_of_ball.argtypes = [POINTER(c_uint64), POINTER(c_uint32), c_uint64,
                                         c_uint32, c_uint64, POINTER(_Params), POINTER(c_uint64)]
        L.or_distance_distribution.argtypes = [POINTER(c_double), c_uint64, POINTER(c_double),
                                               POINTER(c_double), POINTER(c_double)]
        L.or_effective_diameter.argtypes = [POINTER(c_double), c_uint64, c_double, c_int,
                                            POINTER(c_double)]
        L.or_gen_rmat.argtypes = [c_uint32, c_uint32, c_double, c_double, c_double, c_uint64,
                                  c_uint64, ctypes.c_uint, POINTER(_Graph)]
        L.or_counter_digest.restype = c_uint64
        L.or_counter_digest.argtypes = [POINTER(c_uint64), c_uint64, ctypes.c_uint, ctypes.c_uint]
        L.or_csr_digest.restype = c_uint64
        L.or_csr_digest.argtypes = [POINTER(c_uint64), POINTER(c_uint32), c_uint64]
        self.L = L

    # sketch primitives ------------------------------------------------------
    def params(self, b, seed=0, r=5):
        p = _Params()
        if self.L.or_params_make(b, seed, r, ctypes.byref(p)) != 0:
            raise ValueError("invalid sketch parameters")
        return p

    def item_hash(self, item, seed):
        return self.L.or_item_hash(item, seed)

    def counter_of(self, p, items):
        c = np.zeros(p.words, dtype=np.uint64)
        for it in items:
            self.L.or_counter_add(_u64p(c), ctypes.byref(p), int(it))
        return c

    def estimate(self, c, p):
        c = np.ascontiguousarray(c, dtype=np.uint64)
        return self.L.or_counter_estimate(_u64p(c), ctypes.byref(p))

    def read_register(self, c, p, j):
        return self.L.or_read_register(_u64p(c), ctypes.byref(p), j)

    def write_register(self, c, p, j, v):
        self.L.or_write_register(_u64p(c), ctypes.byref(p), j, v)

    def packed_max_into(self, p, dst, src):
        return self.L.or_packed_max_into(ctypes.byref(p), _u64p(dst), _u64p(src))

    def naive_union(self, dst, src, p):
        return self.L.or_naive_union(_u64p(dst), _u64p(src), ctypes.byref(p))

    # graphs -----------------------------------------------------------------
    def _take(self, g: _Graph):
        n, a = g.n, g.arcs
        off = np.ctypeslib.as_array(g.offsets, shape=(n + 1,)).copy()
        succ = (np.ctypeslib.as_array(g.succ, shape=(a,)).copy() if a
                else np.zeros(0, dtype=np.uint32))
        self.L.or_graph_free(ctypes.byref(g))
        return n, off, succ

    def gen_uniform_random(self, n, d, seed):
        g = _Graph()
        if self.L.or_gen_uniform_random(n, d, seed, ctypes.byref(g)) != 0:
            raise ValueError("bad generator arguments")
        return self._take(g)

    def gen_clique_path(self, k, l):
        g = _Graph()
        if self.L.or_gen_clique_path(k, l, ctypes.byref(g)) != 0:
            raise ValueError("bad generator arguments")
        return self._take(g)

    def gen_rmat(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, permute_seed=7,
                 threads=None):
        """BASELINE configs 2/5 R-MAT (hanf_oracle_gen.c), multi-threaded.
        Returns (n, offsets, succ); the arrays own the C buffers (no copy)."""
        g = _Graph()
        rc = self.L.or_gen_rmat(scale, edge_factor, a, b, c, seed, permute_seed,
                                threads or os.cpu_count() or 1, ctypes.byref(g))
        if rc:
            raise (MemoryError if rc == -2 else ValueError)("or_gen_rmat failed")
        return g.n, _owned(self, g, g.offsets, g.n + 1), _owned(self, g, g.succ, g.arcs)

    def counter_digest(self, words, n, W, threads=None):
        """words: a uint64 array, or a ctypes POINTER(c_uint64)."""
        if isinstance(words, np.ndarray):
            w = np.ascontiguousarray(words, dtype=np.uint64)
            assert w.size >= n * W
            words = _u64p(w)
        return int(self.L.or_counter_digest(words, n, W, threads or os.cpu_count() or 1))

    def csr_digest(self, n, offsets, succ):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        succ = np.ascontiguousarray(succ, dtype=np.uint32)
        if succ.size == 0:
            succ = np.zeros(1, dtype=np.uint32)
        return int(self.L.or_csr_digest(_u64p(offsets), _u32p(succ), n))

    def from_edges(self, n, src, dst):
        src = np.ascontiguousarray(src, dtype=np.uint32)
        dst = np.ascontiguousarray(dst, dtype=np.uint32)
        g = _Graph()
        if self.L.or_graph_from_edges(n, _u32p(src), _u32p(dst), src.size, ctypes.byref(g)):
            raise ValueError("arc endpoint out of range")
        return self._take(g)

    def exact_nf(self, n, offsets, succ):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        succ = np.ascontiguousarray(succ, dtype=np.uint32)
        vals = np.zeros(n + 2, dtype=np.uint64)
        ln = c_uint64()
        if self.L.or_exact_nf(_u64p(offsets), _u32p(succ), n, _u64p(vals), vals.size,
                              ctypes.byref(ln)):
            raise RuntimeError("exact_nf capacity")
        return [int(x) for x in vals[:ln.value]]

    def clique_path_nf(self, k, l, t):
        return self.L.or_clique_path_nf(k, l, t)

    def counter_of_ball(self, n, offsets, succ, v, radius, p):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        succ = np.ascontiguousarray(succ, dtype=np.uint32)
        out = np.zeros(p.words, dtype=np.uint64)
        self.L.or_counter_of_ball(_u64p(offsets), _u32p(succ), n, v, radius, ctypes.byref(p),
                                  _u64p(out))
        return out

    # engine -----------------------------------------------------------------
    def engine(self, n, offsets, succ, **cfg):
        return PortEngine(self, n, offsets, succ, **cfg)

    def distance_distribution(self, nf):
        a = np.ascontiguousarray(nf, dtype=np.float64)
        m, v, s = c_double(), c_double(), c_double()
        if self.L.or_distance_distribution(_f64p(a), a.size, ctypes.byref(m), ctypes.byref(v),
                                           ctypes.byref(s)):
            raise ValueError("bad input")
        return m.value, v.value, s.value

    def effective_diameter(self, nf, alpha=0.9, interpolated=False):
        a = np.ascontiguousarray(nf, dtype=np.float64)
        out = c_double()
        if self.L.or_effective_diameter(_f64p(a), a.size, alpha, int(interpolated),
                                        ctypes.byref(out)):
            raise ValueError("bad input")
        return out.value


class _CBuffers:
    """Frees an or_graph's malloc'd arrays when the last view goes."""

    def __init__(self, port, g):
        self.port, self.g = port, g
        self.refs = 0

    def release(self):
        self.refs -= 1
        if self.refs == 0:
            self.port.L.or_graph_free(ctypes.byref(self.g))


class _OwnedArray(np.ndarray):
    def __del__(self):
        owner = getattr(self, "_owner", None)
        if owner is not None:
            self._owner = None
            owner.release()


_owners = {}


def _owned(port, g, ptr, count):
    key = ctypes.addressof(g)
    owner = _owners.get(key)
    if owner is None or owner.g is not g:
        owner = _owners[key] = _CBuffers(port, g)
    if count == 0:
        return np.zeros(0, dtype=np.uint32 if ptr._type_ is c_uint32 else np.uint64)
    arr = np.ctypeslib.as_array(ptr, shape=(int(count),)).view(_OwnedArray)
    arr._owner = owner
    owner.refs += 1
    return arr


class PortEngine:
    """The oracle engine (engine.hpp:68-292 restated in hanf_oracle.c)."""

    def __init__(self, port: Port, n, offsets, succ, **cfg):
        self.port, self.L = port, port.L
        self.n = int(n)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.succ = np.ascontiguousarray(succ, dtype=np.uint32)
        c = _Config()
        self.L.or_config_default(ctypes.byref(c))
        for k, v in cfg.items():
            setattr(c, k, int(v) if k not in ("systolic_threshold", "eps_inc") else float(v))
        st = c_int()
        self.h = self.L.or_engine_create(_u64p(self.offsets), _u32p(self.succ), self.n,
                                         ctypes.byref(c), ctypes.byref(st))
        if not self.h:
            raise ValueError("invalid engine configuration")
        self.words = self.L.or_engine_words(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.or_engine_destroy(self.h)
            self.h = None

    def sum_estimates(self):
        return self.L.or_engine_sum_estimates(self.h)

    def step(self):
        s, m = c_double(), c_uint64()
        self.L.or_engine_step(self.h, ctypes.byref(s), ctypes.byref(m))
        return s.value, m.value

    def counters(self):
        p = self.L.or_engine_counters(self.h)
        return np.ctypeslib.as_array(p, shape=(self.n * self.words,)).copy()

    def iteration(self):
        return self.L.or_engine_iteration(self.h)

    def systolic_active(self):
        return bool(self.L.or_engine_systolic_active(self.h))

    def run(self, cap=None):
        cap = cap or (self.n + 2)
        vals = np.zeros(cap, dtype=np.float64)
        mods = np.zeros(cap, dtype=np.uint64)
        ln = c_uint64()
        rc = self.L.or_engine_run(self.h, _f64p(vals), _u64p(mods), cap, ctypes.byref(ln))
        if rc == 2:
            raise RuntimeError("GuardError: iteration cap exceeded")
        if rc != 0:
            raise RuntimeError(f"oracle run failed ({rc})")
        L = ln.value
        return list(vals[:L]), [int(x) for x in mods[:L]]


# --------------------------------------------------------------------------
# ref: the reference engine itself (through ref_shim.cpp)
# --------------------------------------------------------------------------
class Ref:
    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = ctypes.CDLL(path)
        vp = c_void_p
        L.ref_graph_from_csr.restype = vp
        L.ref_graph_from_csr.argtypes = [c_uint64, POINTER(c_uint64), POINTER(c_uint32)]
        L.ref_gen_uniform_random.restype = vp
        L.ref_gen_uniform_random.argtypes = [c_uint64, c_double, c_uint64]
        L.ref_gen_clique_path.restype = vp
        L.ref_gen_clique_path.argtypes = [c_uint64, c_uint64]
        L.ref_graph_nodes.restype = c_uint64
        L.ref_graph_nodes.argtypes = [vp]
        L.ref_graph_arcs.restype = c_uint64
        L.ref_graph_arcs.argtypes = [vp]
        L.ref_graph_csr.argtypes = [vp, POINTER(c_uint64), POINTER(c_uint32)]
        L.ref_graph_free.argtypes = [vp]
        L.ref_engine_create.restype = vp
        L.ref_engine_create.argtypes = [vp, ctypes.c_uint, ctypes.c_uint, c_uint64,
                                        ctypes.c_uint, c_uint64, c_double, c_int, c_double,
                                        c_uint64, c_int, c_int, POINTER(c_int)]
        L.ref_engine_free.argtypes = [vp]
        L.ref_engine_sum_estimates.restype = c_double
        L.ref_engine_sum_estimates.argtypes = [vp]
        L.ref_engine_step.argtypes = [vp, POINTER(c_double), POINTER(c_uint64)]
        L.ref_engine_timed_step.restype = c_double
        L.ref_engine_timed_step.argtypes = [vp, POINTER(c_double), POINTER(c_uint64)]
        L.ref_engine_counters.restype = POINTER(c_uint64)
        L.ref_engine_counters.argtypes = [vp, POINTER(c_uint64)]
        L.ref_engine_iteration.restype = c_uint64
        L.ref_engine_iteration.argtypes = [vp]
        L.ref_engine_save_counters.argtypes = [vp, ctypes.c_char_p]
        L.ref_engine_systolic_active.argtypes = [vp]
        L.ref_engine_run.argtypes = [vp, POINTER(c_double), POINTER(c_uint64), c_uint64,
                                     POINTER(c_uint64), POINTER(c_double)]
        L.ref_counter_add.argtypes = [POINTER(c_uint64), ctypes.c_uint, ctypes.c_uint, c_uint64,
                                      c_uint64]
        L.ref_counter_estimate.restype = c_double
        L.ref_counter_estimate.argtypes = [POINTER(c_uint64), ctypes.c_uint, ctypes.c_uint]
        L.ref_counter_union.argtypes = [POINTER(c_uint64), POINTER(c_uint64), ctypes.c_uint,
                                        ctypes.c_uint]
        L.ref_distance_distribution.argtypes = [POINTER(c_double), c_uint64, POINTER(c_double),
                                                POINTER(c_double), POINTER(c_double)]
        L.ref_effective_diameter.argtypes = [POINTER(c_double), c_uint64, c_double, c_int,
                                             POINTER(c_double)]
        L.ref_exact_nf.argtypes = [vp, POINTER(c_uint64), c_uint64, POINTER(c_uint64)]
        L.ref_hardware_threads.restype = ctypes.c_uint
        L.ref_graph_from_sorted_csr.restype = vp
        L.ref_graph_from_sorted_csr.argtypes = [c_uint64, POINTER(c_uint64), POINTER(c_uint32)]
        L.ref_engine_step_sample.restype = c_double
        L.ref_engine_step_sample.argtypes = [vp, c_uint64, c_uint64, ctypes.c_uint,
                                             POINTER(c_uint64), POINTER(c_double),
                                             POINTER(c_uint64)]
        L.ref_engine_prefault.argtypes = [vp, ctypes.c_uint]
        L.ref_engine_next_counters.restype = POINTER(c_uint64)
        L.ref_engine_next_counters.argtypes = [vp, POINTER(c_uint64)]
        self.L = L

    def graph(self, n, offsets, succ):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        succ = np.ascontiguousarray(succ, dtype=np.uint32)
        return RefGraph(self, self.L.ref_graph_from_csr(n, _u64p(offsets), _u32p(succ)))

    def graph_sorted(self, n, offsets, succ):
        """hyperanf::Graph from a sorted, deduplicated CSR in O(a): the same
        object Graph::from_edges builds, without its std::sort."""
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        succ = np.ascontiguousarray(succ, dtype=np.uint32)
        if succ.size == 0:
            succ = np.zeros(1, dtype=np.uint32)
        h = self.L.ref_graph_from_sorted_csr(n, _u64p(offsets), _u32p(succ))
        if not h:
            raise ValueError("CSR rows are not sorted / deduplicated / in range")
        return RefGraph(self, h)

    def gen_uniform_random(self, n, d, seed):
        return RefGraph(self, self.L.ref_gen_uniform_random(n, d, seed))

    def gen_clique_path(self, k, l):
        return RefGraph(self, self.L.ref_gen_clique_path(k, l))

    def engine(self, graph, bucket_bits=7, register_bits=0, seed=0, threads=1, task_size=0,
               systolic_threshold=0.25, termination=0, eps_inc=0.0, max_iterations=0,
               track_modified=True, use_systolic=True):
        st = c_int()
        h = self.L.ref_engine_create(graph.h, bucket_bits, register_bits, seed, threads,
                                     task_size, systolic_threshold, termination, eps_inc,
                                     max_iterations, int(track_modified), int(use_systolic),
                                     ctypes.byref(st))
        if not h:
            raise ValueError(f"reference engine rejected the config ({st.value})")
        return RefEngine(self, h, graph)

    def counter_estimate(self, words, b, r=5):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        return self.L.ref_counter_estimate(_u64p(w), b, r)

    def exact_nf(self, graph):
        cap = graph.n + 2
        vals = np.zeros(cap, dtype=np.uint64)
        ln = c_uint64()
        rc = self.L.ref_exact_nf(graph.h, _u64p(vals), cap, ctypes.byref(ln))
        if rc:
            raise RuntimeError(f"exact_nf failed ({rc})")
        return [int(x) for x in vals[:ln.value]]

    def distance_distribution(self, nf):
        a = np.ascontiguousarray(nf, dtype=np.float64)
        m, v, s = c_double(), c_double(), c_double()
        if self.L.ref_distance_distribution(_f64p(a), a.size, ctypes.byref(m), ctypes.byref(v),
                                            ctypes.byref(s)):
            raise ValueError("bad input")
        return m.value, v.value, s.value

    def effective_diameter(self, nf, alpha=0.9, interpolated=False):
        a = np.ascontiguousarray(nf, dtype=np.float64)
        out = c_double()
        if self.L.ref_effective_diameter(_f64p(a), a.size, alpha, int(interpolated),
                                         ctypes.byref(out)):
            raise ValueError("bad input")
        return out.value

    def hardware_threads(self):
        return self.L.ref_hardware_threads()


class RefGraph:
    def __init__(self, ref: Ref, h):
        if not h:
            raise ValueError("reference graph construction failed")
        self.ref, self.h = ref, h
        self.n = ref.L.ref_graph_nodes(h)
        self.arcs = ref.L.ref_graph_arcs(h)

    def csr(self):
        off = np.zeros(self.n + 1, dtype=np.uint64)
        succ = np.zeros(max(self.arcs, 1), dtype=np.uint32)
        self.ref.L.ref_graph_csr(self.h, _u64p(off), _u32p(succ))
        return off, succ[:self.arcs]

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.ref_graph_free(self.h)
            self.h = None


class RefEngine:
    def __init__(self, ref: Ref, h, graph: RefGraph):
        self.ref, self.L, self.h, self.graph = ref, ref.L, h, graph

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_engine_free(self.h)
            self.h = None

    def sum_estimates(self):
        return self.L.ref_engine_sum_estimates(self.h)

    def step(self):
        s, m = c_double(), c_uint64()
        self.L.ref_engine_step(self.h, ctypes.byref(s), ctypes.byref(m))
        return s.value, m.value

    def timed_step(self):
        s, m = c_double(), c_uint64()
        secs = self.L.ref_engine_timed_step(self.h, ctypes.byref(s), ctypes.byref(m))
        return secs, s.value, m.value

    def counters(self):
        wc = c_uint64()
        p = self.L.ref_engine_counters(self.h, ctypes.byref(wc))
        return np.ctypeslib.as_array(p, shape=(wc.value,)).copy() if wc.value else \
            np.zeros(0, dtype=np.uint64)

    def iteration(self):
        return self.L.ref_engine_iteration(self.h)

    def step_sample(self, lo, hi, threads):
        """NfEngine::step's per-node body over [lo, hi) plus the block
        re-sum (ref_shim.cpp ref_engine_step_sample); no swap.
        Returns (seconds, arcs, block sum, changed)."""
        arcs, s, ch = c_uint64(), c_double(), c_uint64()
        secs = self.L.ref_engine_step_sample(self.h, lo, hi, threads, ctypes.byref(arcs),
                                             ctypes.byref(s), ctypes.byref(ch))
        return secs, arcs.value, s.value, ch.value

    def counters_ptr(self):
        """(pointer, word count) of the engine's current counters, no copy."""
        wc = c_uint64()
        p = self.L.ref_engine_counters(self.h, ctypes.byref(wc))
        return p, wc.value

    def prefault(self, threads):
        """Allocate and touch next_ (ref_shim.cpp ref_engine_prefault)."""
        self.L.ref_engine_prefault(self.h, threads)

    def next_counters(self):
        wc = c_uint64()
        p = self.L.ref_engine_next_counters(self.h, ctypes.byref(wc))
        return np.ctypeslib.as_array(p, shape=(wc.value,)).copy() if wc.value else \
            np.zeros(0, dtype=np.uint64)

    def save_counters(self, path):
        """The reference's own HCA1 writer (hll.hpp:275-286)."""
        assert self.L.ref_engine_save_counters(self.h, str(path).encode()) == 0

    def systolic_active(self):
        return bool(self.L.ref_engine_systolic_active(self.h))

    def run(self, cap=None):
        cap = cap or (self.graph.n + 2)
        vals = np.zeros(cap, dtype=np.float64)
        mods = np.zeros(cap, dtype=np.uint64)
        ln, wall = c_uint64(), c_double()
        rc = self.L.ref_engine_run(self.h, _f64p(vals), _u64p(mods), cap, ctypes.byref(ln),
                                   ctypes.byref(wall))
        if rc == 2:
            raise RuntimeError("GuardError")
        if rc:
            raise RuntimeError(f"reference run failed ({rc})")
        L = ln.value
        return list(vals[:L]), [int(x) for x in mods[:L]], wall.value


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def have_ref() -> bool:
    return os.path.exists(REF_PATH)
