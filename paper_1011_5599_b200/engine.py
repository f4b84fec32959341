"""The HyperANF engine: Python mirror of ``hyperanf::NfEngine`` (engine.hpp).

Every method is a thin call through the C-ABI of libhanf.so, whose union,
estimate and reduction kernels run on the B200.  Names, argument meaning and
error behaviour follow the reference:

    EngineConfig      engine.hpp:32-46
    IterationReport   engine.hpp:48-51
    NfEstimate        engine.hpp:53-66
    NfEngine          engine.hpp:68-292
    estimate_nf       engine.hpp:295-298
    SketchParams      hll.hpp:36-70
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
from ctypes import POINTER, c_double, c_int32, c_uint64, c_void_p
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _lib
from ._lib import check, lib
from .graph import Graph


class Termination(enum.IntEnum):
    stabilisation = 0
    threshold = 1


@dataclass
class EngineConfig:
    bucket_bits: int = 7
    register_bits: int = 0          # 0: 5 below 2^32 nodes, 6 otherwise
    seed: int = 0
    threads: int = 1                # CPU scheduling knob (accepted, no effect)
    task_size: int = 0              # CPU scheduling knob (accepted, no effect)
    systolic_threshold: float = 0.25
    termination: Termination = Termination.stabilisation
    eps_inc: float = 0.0
    max_iterations: int = 0         # 0: n + 1
    spill_to_disk: bool = False     # accepted; HBM holds both generations
    track_modified: bool = True
    use_systolic: bool = True
    # B200 options: never change a result bit
    device: int = 0
    exact_sum: bool = True          # N(t) total in the reference's summation order
    shard_begin: int = 0
    shard_end: int = 0
    shard_count: int = 0            # peer-push shards: allows relabelled shards
    expected_runs: int = 0          # runs planned on this engine (multirun sets it):
                                    # from 20, large engines build their source-blocked
                                    # dense sweeps at create (hanf_block_stats)
    # several GPUs of this process, one node-range shard each (repeats
    # allowed): the engine drives them all (hanf_create_multi)
    devices: tuple = ()

    def to_c(self) -> _lib.Config:
        c = _lib.Config()
        check(lib().hanf_config_init(ctypes.byref(c)))
        c.bucket_bits = self.bucket_bits
        c.register_bits = self.register_bits
        c.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        c.threads = self.threads
        c.task_size = self.task_size
        c.systolic_threshold = self.systolic_threshold
        c.termination = int(self.termination)
        c.eps_inc = self.eps_inc
        c.max_iterations = self.max_iterations
        c.spill_to_disk = int(self.spill_to_disk)
        c.track_modified = int(self.track_modified)
        c.use_systolic = int(self.use_systolic)
        c.device = self.device
        c.exact_sum = int(self.exact_sum)
        c.shard_begin = self.shard_begin
        c.shard_end = self.shard_end
        c.shard_count = self.shard_count
        c.expected_runs = max(0, min(int(self.expected_runs), 0xFFFFFFFF))
        return c


@dataclass
class IterationReport:
    sum: float = 0.0
    modified: int = 0


@dataclass
class NfEstimate:
    n: int = 0
    m: int = 0
    seed: int = 0
    termination: Termination = Termination.stabilisation
    values: List[float] = field(default_factory=list)
    modified: List[int] = field(default_factory=list)
    wall_seconds: float = 0.0
    exact: bool = False

    def iterations(self) -> int:
        return 0 if not self.values else len(self.values) - 1


@dataclass
class SketchParams:
    bucket_bits: int = 7
    registers: int = 128
    register_bits: int = 5
    alpha: float = 0.0
    seed: int = 0
    words: int = 10

    @staticmethod
    def make(bucket_bits: int, seed: int, register_bits: int = 5) -> "SketchParams":
        """hll.hpp:43-56 (raises ValueError like std::invalid_argument)."""
        p = _lib.SketchParamsC()
        check(lib().hanf_sketch_params_make(bucket_bits, seed & 0xFFFFFFFFFFFFFFFF,
                                            register_bits, ctypes.byref(p)))
        return SketchParams._from_c(p)

    @staticmethod
    def _from_c(p: _lib.SketchParamsC) -> "SketchParams":
        return SketchParams(p.bucket_bits, p.registers, p.register_bits, p.alpha, p.seed,
                            p.words_per_counter)

    def words_per_counter(self) -> int:
        return self.words

    def max_register_value(self) -> int:
        return (1 << self.register_bits) - 1


class NfEngine:
    """Neighbourhood-function estimator over one HLL counter per node.

    The engine keeps its own copy of the graph in HBM (the reference keeps
    a non-owning pointer; the caller's Graph may be dropped after
    construction here)."""

    def __init__(self, graph: Graph, cfg: EngineConfig = None):
        cfg = cfg or EngineConfig()
        self._cfg = dataclasses.replace(cfg)  # (reseed / restore update the engine's copy only)
        self._graph = graph
        self._h = c_void_p()
        view = graph.view()
        ccfg = cfg.to_c()
        if cfg.devices:
            devs = (c_int32 * len(cfg.devices))(*cfg.devices)
            check(lib().hanf_create_multi(ctypes.byref(view), ctypes.byref(ccfg), devs,
                                          len(cfg.devices), ctypes.byref(self._h)))
        else:
            check(lib().hanf_create(ctypes.byref(view), ctypes.byref(ccfg),
                                    ctypes.byref(self._h)))
        p = _lib.SketchParamsC()
        check(lib().hanf_params(self._h, ctypes.byref(p)))
        self._params = SketchParams._from_c(p)

    def close(self) -> None:
        if self._h:
            lib().hanf_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- reference surface (engine.hpp:92-96) ---------------------------------
    def params(self) -> SketchParams:
        return self._params

    def config(self) -> EngineConfig:
        return self._cfg

    def iteration(self) -> int:
        t = c_uint64()
        check(lib().hanf_iteration(self._h, ctypes.byref(t)))
        return t.value

    def systolic_active(self) -> bool:
        a = c_int32()
        check(lib().hanf_systolic_active(self._h, ctypes.byref(a)))
        return bool(a.value)

    def counters(self, first: int = 0, count: int = None) -> np.ndarray:
        """CounterArray::data() (hll.hpp:224-226): u64[count * W] in the
        reference packing, copied from HBM."""
        n = self._graph.num_nodes()
        if count is None:
            count = n - first
        out = np.empty(max(count, 0) * self._params.words, dtype=np.uint64)
        check(lib().hanf_read_counters(self._h, first, count,
                                       out.ctypes.data_as(POINTER(c_uint64))))
        return out

    def counter(self, i: int) -> np.ndarray:
        """CounterArray::counter(i) (hll.hpp:196-205); IndexError past n."""
        return self.counters(i, 1)

    def sum_estimates(self) -> float:
        s = c_double()
        check(lib().hanf_sum_estimates(self._h, ctypes.byref(s)))
        return s.value

    def step(self) -> IterationReport:
        r = _lib.IterationReportC()
        check(lib().hanf_step(self._h, ctypes.byref(r)))
        return IterationReport(r.sum, r.modified)

    def step_launch(self) -> None:
        """hanf_step_launch: enqueue one step on stream() and return."""
        check(lib().hanf_step_launch(self._h))

    def step_complete(self) -> IterationReport:
        """hanf_step_complete: wait for the launched step, report it."""
        r = _lib.IterationReportC()
        check(lib().hanf_step_complete(self._h, ctypes.byref(r)))
        return IterationReport(r.sum, r.modified)

    def run_to_stabilisation(self) -> NfEstimate:
        """engine.hpp:233-275: N(0..T), clamped non-decreasing; the
        stabilising no-change iteration is not recorded."""
        n = self._graph.num_nodes()
        cap = 64
        vals = np.empty(cap, dtype=np.float64)
        mods = np.empty(cap, dtype=np.uint64)
        length = c_uint64()
        wall = c_double()
        st = lib().hanf_run_to_stabilisation(
            self._h, vals.ctypes.data_as(POINTER(c_double)),
            mods.ctypes.data_as(POINTER(c_uint64)), cap, ctypes.byref(length),
            ctypes.byref(wall))
        if st == _lib.CAPACITY:
            cap = length.value
            vals = np.empty(cap, dtype=np.float64)
            mods = np.empty(cap, dtype=np.uint64)
            st = lib().hanf_last_result(self._h, vals.ctypes.data_as(POINTER(c_double)),
                                        mods.ctypes.data_as(POINTER(c_uint64)), cap,
                                        ctypes.byref(length))
        check(st)
        L = length.value
        return NfEstimate(n=n, m=self._params.registers, seed=self._params.seed,
                          termination=self._cfg.termination,
                          values=[float(x) for x in vals[:L]],
                          modified=[int(x) for x in mods[:L]], wall_seconds=wall.value)

    # -- B200 plumbing ------------------------------------------------------------
    def reset(self) -> None:
        """Re-seed and rewind to iteration 0 (no graph re-upload)."""
        check(lib().hanf_reset(self._h))

    def save_counters(self, path) -> None:
        """hll.hpp:275-286: the current counters as an HCA1 snapshot, byte
        for byte the reference's save_counters output."""
        check(lib().hanf_save_counters(self._h, str(path).encode()))

    def restore_counters(self, path, iteration: int = 0) -> None:
        """Resume from an HCA1 snapshot (hll.hpp:288-303) taken at
        `iteration`: both generations hold it, every counter counts as
        modified, N(t) is re-summed; the snapshot's seed is adopted."""
        check(lib().hanf_restore_counters(self._h, str(path).encode(), iteration))
        p = _lib.SketchParamsC()
        check(lib().hanf_params(self._h, ctypes.byref(p)))
        self._params = SketchParams._from_c(p)
        self._cfg.seed = self._params.seed

    def reseed(self, seed: int) -> None:
        """reset() under another HLL seed (hanf_reseed): the next run of a
        multi-seed experiment without re-uploading the graph."""
        check(lib().hanf_reseed(self._h, seed & 0xFFFFFFFFFFFFFFFF))
        self._cfg.seed = seed
        p = _lib.SketchParamsC()
        check(lib().hanf_params(self._h, ctypes.byref(p)))
        self._params = SketchParams._from_c(p)

    def stream(self) -> int:
        s = c_void_p()
        check(lib().hanf_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def launch_count(self) -> int:
        c = c_uint64()
        check(lib().hanf_launch_count(self._h, ctypes.byref(c)))
        return c.value

    def block_stats(self):
        """hanf_block_stats: (items, arcs they cover) of the source-blocked
        dense sweeps, (0, 0) when the engine does not use them."""
        items, arcs = c_uint64(), c_uint64()
        check(lib().hanf_block_stats(self._h, ctypes.byref(items), ctypes.byref(arcs)))
        return int(items.value), int(arcs.value)

    def set_timing(self, enable: bool = True) -> None:
        """CUDA-event phase timing on the engine stream (resets the totals)."""
        check(lib().hanf_set_timing(self._h, int(enable)))

    def timing(self) -> dict:
        u, e, r, n = c_double(), c_double(), c_double(), c_uint64()
        check(lib().hanf_timing(self._h, ctypes.byref(u), ctypes.byref(e), ctypes.byref(r),
                                ctypes.byref(n)))
        return {"union_ms": u.value, "estimate_ms": e.value, "reduce_ms": r.value,
                "steps": n.value}

    def device_buffers(self) -> _lib.BuffersC:
        b = _lib.BuffersC()
        check(lib().hanf_device_buffers(self._h, ctypes.byref(b)))
        return b

    def shard_compute(self) -> None:
        check(lib().hanf_shard_compute(self._h))

    def shard_export(self) -> bytes:
        """hanf_shard_export: this shard's exchange arena as bytes (to be
        all-gathered and handed to every rank's shard_attach)."""
        d = _lib.ShardPeerC()
        check(lib().hanf_shard_export(self._h, ctypes.byref(d)))
        return ctypes.string_at(ctypes.addressof(d), ctypes.sizeof(d))

    def shard_attach(self, peers, self_index: int) -> None:
        """hanf_shard_attach: peer-push exchange with the ranks' exports."""
        arr = (_lib.ShardPeerC * len(peers))()
        for i, raw in enumerate(peers):
            ctypes.memmove(ctypes.addressof(arr[i]), bytes(raw), ctypes.sizeof(_lib.ShardPeerC))
        check(lib().hanf_shard_attach(self._h, arr, len(peers), self_index))

    def shard_attach_local(self, peers, self_index: int) -> None:
        """hanf_shard_attach_local: peer-push between engines of this process."""
        arr = (c_void_p * len(peers))(*[p._h.value for p in peers])
        check(lib().hanf_shard_attach_local(self._h, arr, len(peers), self_index))

    def shard_detach(self) -> None:
        check(lib().hanf_shard_detach(self._h))

    def shard_reduce(self) -> None:
        """hanf_shard_reduce: relabelled peer-push shards re-sum one slice of
        the block sums each (between two barriers); a no-op otherwise."""
        check(lib().hanf_shard_reduce(self._h))

    def shard_push_stats(self):
        """hanf_shard_push_stats: (rows of this shard the last committed step
        changed, row stores those changes pushed to peers)."""
        changed, pushed = c_uint64(), c_uint64()
        check(lib().hanf_shard_push_stats(self._h, ctypes.byref(changed), ctypes.byref(pushed)))
        return int(changed.value), int(pushed.value)

    def shard_commit(self) -> IterationReport:
        r = _lib.IterationReportC()
        check(lib().hanf_shard_commit(self._h, ctypes.byref(r)))
        return IterationReport(r.sum, r.modified)


def estimate_nf(g: Graph, cfg: EngineConfig = None) -> NfEstimate:
    """engine.hpp:295-298: seed counters, run, return the estimate."""
    with NfEngine(g, cfg or EngineConfig()) as engine:
        return engine.run_to_stabilisation()


@dataclass
class ExactNf:
    """oracle.hpp:24-35: values[t] = ordered pairs (x, y) with d(x, y) <= t."""
    n: int = 0
    values: List[int] = field(default_factory=list)

    def diameter(self) -> int:
        return 0 if not self.values else len(self.values) - 1

    def as_doubles(self) -> List[float]:
        return [float(v) for v in self.values]


def exact_nf(g: Graph, device: int = 0, max_nodes: int = 1_000_000,
             max_work: int = 100_000_000_000) -> ExactNf:
    """oracle.hpp:38-104 (exact NF, same guard -> GuardError), computed on
    the GPU as bitset balls (hanf_exact.cu) instead of all-pairs BFS."""
    view = g.view()
    cap = 64
    while True:
        vals = np.empty(cap, dtype=np.uint64)
        length = c_uint64()
        st = lib().hanf_exact_nf(ctypes.byref(view), device, max_nodes, max_work,
                                 vals.ctypes.data_as(POINTER(c_uint64)), cap,
                                 ctypes.byref(length))
        if st == _lib.CAPACITY:
            cap = length.value
            continue
        check(st)
        return ExactNf(n=g.num_nodes(), values=[int(x) for x in vals[:length.value]])


def _run_batch(g: Graph, cfg: EngineConfig, seeds) -> List[NfEstimate]:
    """len(seeds) in {2, 4, 8} runs in one batched engine (hanf_create_batch)."""
    import time
    k = len(seeds)
    h = c_void_p()
    view = g.view()
    ccfg = cfg.to_c()
    sarr = (c_uint64 * k)(*[s_ & 0xFFFFFFFFFFFFFFFF for s_ in seeds])
    check(lib().hanf_create_batch(ctypes.byref(view), ctypes.byref(ccfg), sarr, k,
                                  ctypes.byref(h)))
    try:
        p = _lib.SketchParamsC()
        check(lib().hanf_params(h, ctypes.byref(p)))
        cap = 64
        while True:
            vals = np.empty(k * cap, dtype=np.float64)
            mods = np.empty(k * cap, dtype=np.uint64)
            lens = (c_uint64 * k)()
            t0 = time.perf_counter()
            st = lib().hanf_run_batch(h, vals.ctypes.data_as(POINTER(c_double)),
                                      mods.ctypes.data_as(POINTER(c_uint64)), cap, lens)
            wall = time.perf_counter() - t0
            if st == _lib.CAPACITY:
                cap = max(lens)
                check(lib().hanf_reset(h))
                continue
            check(st)
            break
        return [NfEstimate(n=g.num_nodes(), m=p.registers, seed=seeds[i],
                           termination=cfg.termination,
                           values=[float(x) for x in vals[i * cap:i * cap + lens[i]]],
                           modified=[int(x) for x in mods[i * cap:i * cap + lens[i]]],
                           wall_seconds=wall / k) for i in range(k)]
    finally:
        lib().hanf_destroy(h)


def multirun(g: Graph, cfg: EngineConfig = None, runs: int = 10, base_seed: int = None,
             batch: int = 1):
    """The reference's multirun (main.cpp:263-283): estimate_nf for seeds
    base_seed + i, i < runs (base_seed defaults to cfg.seed).  batch = 1:
    one engine re-seeded per run (the graph is uploaded and laid out once);
    batch in {2, 4, 8}: that many runs at a time in one batched engine
    (hanf_create_batch).  Bit-identical either way; aggregate with
    stats.aggregate_runs."""
    import dataclasses
    cfg = dataclasses.replace(cfg) if cfg is not None else EngineConfig()
    base = cfg.seed if base_seed is None else base_seed
    out = []
    if runs <= 0:
        return out
    if batch > 1:
        i = 0
        while i < runs:
            k = next(b for b in (8, 4, 2, 1) if b <= min(batch, runs - i))
            seeds = [base + i + j for j in range(k)]
            if k == 1:
                out.append(estimate_nf(g, dataclasses.replace(cfg, seed=seeds[0])))
            else:
                out.extend(_run_batch(g, cfg, seeds))
            i += k
        return out
    cfg.seed = base
    if not cfg.expected_runs:
        cfg.expected_runs = runs  # the engine may schedule for the whole multi-run
    with NfEngine(g, cfg) as engine:
        for i in range(runs):
            if i:
                engine.reseed(base + i)
            out.append(engine.run_to_stabilisation())
    return out
