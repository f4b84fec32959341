"""CPU-side checks of the drop-in boundary (include/hanf.h, libhanf.so):
the library loads and exports every declared entry point; configuration
errors map to the reference's exception types; graph construction,
generators, HBG1 I/O and the statistics match the reference / oracle."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hanf.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(hanf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(hanf):
    lib = ctypes.CDLL(hanf.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_config_defaults_mirror_engineconfig(hanf):
    """EngineConfig defaults (engine.hpp:32-46)."""
    from paper_1011_5599_b200 import _lib
    c = _lib.Config()
    assert hanf.lib().hanf_config_init(ctypes.byref(c)) == 0
    assert (c.bucket_bits, c.register_bits, c.seed, c.threads, c.task_size) == (7, 0, 0, 1, 0)
    assert (c.systolic_threshold, c.termination, c.eps_inc, c.max_iterations) == (0.25, 0, 0.0, 0)
    assert (c.spill_to_disk, c.track_modified, c.use_systolic) == (0, 1, 1)
    assert (c.exact_sum, c.shard_begin, c.shard_end) == (1, 0, 0)
    d = hanf.EngineConfig()
    assert (d.bucket_bits, d.register_bits, d.systolic_threshold, d.exact_sum) == (7, 0, 0.25, True)


def test_sketch_params_validation(hanf, port):
    """SketchParams::make (hll.hpp:43-56): b in [4, 20], r in [5, 8]."""
    for b, r in [(3, 5), (21, 5), (7, 4), (7, 9)]:
        with pytest.raises(ValueError):
            hanf.SketchParams.make(b, 0, r)
    for b in range(4, 21):
        for r in range(5, 9):
            p = hanf.SketchParams.make(b, 11, r)
            q = port.params(b, 11, r)
            assert (p.registers, p.words, p.alpha) == (q.registers, q.words, q.alpha)
    # words_per_counter examples of test_hll.cpp:31-42
    assert hanf.SketchParams.make(4, 0).words == 2
    assert hanf.SketchParams.make(7, 0).words == 10
    assert hanf.SketchParams.make(8, 0, 6).words == 24


def test_engine_config_errors_are_invalid_argument(hanf):
    """engine.hpp:71-74 (std::invalid_argument) is raised before any device
    work, so it is checked here without a GPU."""
    g = hanf.Graph.from_edges(1, [])
    with pytest.raises(ValueError, match="systolic threshold"):
        hanf.NfEngine(g, hanf.EngineConfig(systolic_threshold=0.0))
    with pytest.raises(ValueError, match="systolic threshold"):
        hanf.NfEngine(g, hanf.EngineConfig(systolic_threshold=1.5))
    with pytest.raises(ValueError, match="eps_inc"):
        hanf.NfEngine(g, hanf.EngineConfig(termination=hanf.Termination.threshold))
    with pytest.raises(ValueError, match="bucket bits"):
        hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=3))
    with pytest.raises(ValueError, match="register width"):
        hanf.NfEngine(g, hanf.EngineConfig(register_bits=9))
    with pytest.raises(ValueError, match="shard"):
        hanf.NfEngine(hanf.gen_uniform_random(200, 3, 1), hanf.EngineConfig(shard_begin=10, shard_end=100))


def test_graph_from_edges(hanf, port):
    """Graph::from_edges (graph.hpp:29-44): sorted rows, duplicates collapsed,
    self-loops kept, endpoints checked."""
    edges = [(3, 1), (0, 2), (3, 1), (2, 2), (0, 1), (3, 0)]
    g = hanf.Graph.from_edges(4, edges)
    n, off, succ = port.from_edges(4, [e[0] for e in edges], [e[1] for e in edges])
    assert np.array_equal(g.offsets(), off) and np.array_equal(g.arcs(), succ)
    assert list(g.successors(3)) == [0, 1] and list(g.successors(2)) == [2]
    with pytest.raises(ValueError):
        hanf.Graph.from_edges(3, [(0, 3)])
    empty = hanf.Graph.from_edges(0, [])
    assert empty.num_nodes() == 0 and empty.num_arcs() == 0


def test_reference_generators_bit_exact(hanf, ref):
    for n, d, seed in [(60, 3, 21), (1000, 8, 4242), (7, 6, 1), (1, 0, 3)]:
        g = hanf.gen_uniform_random(n, d, seed)
        off, succ = ref.gen_uniform_random(n, d, seed).csr()
        assert np.array_equal(g.offsets(), off) and np.array_equal(g.arcs(), succ)
    for k, l in [(1, 1), (4, 3), (260, 10)]:
        g = hanf.gen_clique_path(k, l)
        off, succ = ref.gen_clique_path(k, l).csr()
        assert np.array_equal(g.offsets(), off) and np.array_equal(g.arcs(), succ)
    with pytest.raises(ValueError):
        hanf.gen_uniform_random(5, 5, 1)
    with pytest.raises(ValueError):
        hanf.gen_clique_path(0, 3)


def test_transpose(hanf, port):
    from oracle import _Graph
    g = hanf.gen_uniform_random(300, 4, 9)
    t = hanf.transpose(g)
    src = _Graph(g.num_nodes(), g.num_arcs(), g.offsets().ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                 g.arcs().ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    dst = _Graph()
    port.L.or_graph_transpose(ctypes.byref(src), ctypes.byref(dst))
    n, off, succ = port._take(dst)
    assert np.array_equal(t.offsets(), off) and np.array_equal(t.arcs(), succ)


def _check_csr(g, self_loops=False):
    off, arcs = g.offsets(), g.arcs()
    assert off[0] == 0 and off[-1] == arcs.size and np.all(np.diff(off.astype(np.int64)) >= 0)
    assert arcs.size == 0 or arcs.max() < g.num_nodes()
    src = np.repeat(np.arange(g.num_nodes()), np.diff(off.astype(np.int64)))
    key = src.astype(np.uint64) << np.uint64(32) | arcs.astype(np.uint64)
    assert np.all(np.diff(key.astype(np.int64)) > 0), "rows sorted and deduplicated"
    if not self_loops:
        assert not np.any(src == arcs)


def test_synthetic_generators(hanf):
    """BASELINE config generators: deterministic, CSR-clean, expected sizes."""
    er = hanf.gen_erdos_renyi(4096, 8.0, 1)
    _check_csr(er)
    assert abs(er.num_arcs() / 4096 - 8.0) < 0.4
    assert er == hanf.gen_erdos_renyi(4096, 8.0, 1)
    rm = hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 1, 7)
    _check_csr(rm)
    assert 0.75 * 16 * 4096 < rm.num_arcs() < 16 * 4096  # duplicates removed
    assert rm == hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 1, 7)
    assert rm != hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 1, 8)
    cp = hanf.gen_copying(1 << 14, 2.1, 20.0, 5000, 0.6, 1 << 12, 3)
    _check_csr(cp)
    deg = np.diff(cp.offsets().astype(np.int64))
    assert deg.max() <= 5000 and 14 < deg.mean() < 22
    ba = hanf.gen_barabasi_albert(1 << 12, 10, 4, 11)
    _check_csr(ba)
    assert np.array_equal(ba.offsets(), hanf.transpose(ba).offsets()), "symmetric"
    assert abs(ba.num_arcs() / (2 * 10 * 4096) - 1.0) < 0.05


def test_hbg1_roundtrip(hanf, tmp_path):
    """HBG1 cache (graph.hpp:178-218, FORMATS.md:13-23)."""
    g = hanf.gen_uniform_random(500, 5, 3)
    path = str(tmp_path / "g.hbg")
    hanf.save_csr(g, path)
    with open(path, "rb") as f:
        head = f.read(20)
    assert head[:4] == b"HBG1"
    assert int.from_bytes(head[4:12], "little") == 500
    assert int.from_bytes(head[12:20], "little") == g.num_arcs()
    assert os.path.getsize(path) == 20 + 8 * 501 + 4 * g.num_arcs()
    assert hanf.load_csr(path) == g
    with open(path, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(hanf.ParseError):
        hanf.load_csr(path)
    with pytest.raises(hanf.IoError):
        hanf.load_csr(str(tmp_path / "missing.hbg"))


def test_stats_match_reference(hanf, port, ref):
    """stats.hpp:33-77 (shared C++ implementation in libhanf.so)."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        L = int(rng.integers(1, 30))
        nf = np.cumsum(rng.random(L) * 1e6 + 1.0)
        d = hanf.distance_distribution(nf)
        assert (d.mean, d.variance, d.spid) == ref.distance_distribution(nf)
        assert (d.mean, d.variance, d.spid) == port.distance_distribution(nf)
        for a in (0.5, 0.9, 1.0):
            for interp in (False, True):
                assert hanf.effective_diameter(nf, a, interp) == ref.effective_diameter(nf, a, interp)
    with pytest.raises(ValueError):
        hanf.effective_diameter([], 0.9)
    with pytest.raises(ValueError):
        hanf.effective_diameter([1.0, 2.0], 0.0)
    with pytest.raises(ValueError):
        hanf.cdf_from_nf([0.0, 0.0])


def test_precision_calculators(hanf):
    """acceptance.cpp:315-338 (test_output.txt:17): quoted values."""
    sig3 = lambda a, q: abs(a - q) <= 0.5e-2 * abs(q) + 1e-15  # noqa: E731
    assert sig3(hanf.precision_from_m(256).eta, 0.0662)
    assert sig3(hanf.precision_from_m(128).eta, 0.0937)
    from paper_1011_5599_b200.stats import PrecisionSpec
    assert sig3(PrecisionSpec.ksigma_confidence(2.0), 0.889)
    assert sig3(PrecisionSpec.ksigma_confidence(3.0), 0.951)
    assert sig3(hanf.precision_from_eta(0.0937).memory_gib(1_000_000_000), 74.5)
    with pytest.raises(ValueError):
        hanf.precision_from_m(100)


def test_diameter_interval_and_aggregate(hanf):
    nf = [10.0, 50.0, 90.0, 99.0, 100.0]
    iv = hanf.diameter_interval(nf, 0.9, 0.01, 0.05)
    assert iv.lo == 1 and iv.hi == 3 and iv.confidence == pytest.approx(0.85)
    iv = hanf.diameter_interval(nf, 0.99, 0.01, 0.05)
    assert iv.hi is None and "undefined" in iv.note
    runs = [hanf.NfEstimate(n=5, m=16, seed=s, values=v) for s, v in
            enumerate([[5.0, 10.0, 20.0], [5.0, 12.0, 20.0, 21.0]])]
    rep = hanf.aggregate_runs(runs)
    assert rep.mean_nf == [5.0, 11.0, 20.0, 20.5]
    assert len(rep.per_run) == 2 and rep.stddev.spid >= 0.0
    with pytest.raises(ValueError):
        hanf.aggregate_runs(runs[:1])


def test_create_multi_validates_before_device_work(hanf):
    """hanf_create_multi: device count in [1, 8] and no caller-made shard
    range; rejected with HANF_INVALID_ARGUMENT before any device call."""
    from paper_1011_5599_b200 import _lib
    g = hanf.gen_uniform_random(100, 3, 1)
    view = g.view()
    for count, shard in [(0, 0), (9, 0), (2, 64)]:
        cfg = hanf.EngineConfig(bucket_bits=6, shard_begin=shard, shard_end=2 * shard).to_c()
        devs = (ctypes.c_int32 * 9)(*([0] * 9))
        h = ctypes.c_void_p()
        st = hanf.lib().hanf_create_multi(ctypes.byref(view), ctypes.byref(cfg), devs, count,
                                          ctypes.byref(h))
        assert st == _lib.INVALID_ARGUMENT and not h.value
