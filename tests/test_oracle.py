"""Pins the CPU oracle (oracle/hanf_oracle.c, the checker of the GPU engine)
against the reference: the golden fixtures made from the reference engine
(tests/golden/make_golden.py), the reference's own known answers, and the
reference engine itself run live (oracle/_ref) where it is built."""
from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import graph_of


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_sha(g):
    return sha(np.concatenate([g.offsets().view(np.uint8), g.arcs().view(np.uint8)]))


def test_generators_match_golden(hanf, traces):
    """gen_uniform_random / gen_clique_path (graph.hpp:238-285) reproduce the
    reference's graphs bit for bit; the synthetic R-MAT is pinned too."""
    for case in traces:
        g = graph_of(hanf, case["graph"])
        assert (g.num_nodes(), g.num_arcs()) == (case["n"], case["arcs"]), case["name"]
        assert csr_sha(g) == case["csr_sha256"], case["name"]


@pytest.mark.parametrize("idx", range(28))
def test_port_engine_matches_reference_trace(hanf, port, traces, idx):
    """Lockstep NfEngine::step (engine.hpp:122-228): counters, N(t) and the
    modified count after every iteration, the systolic flag, the
    run_to_stabilisation output and the derived statistics."""
    if idx >= len(traces):
        pytest.skip("fewer golden cases")
    case = traces[idx]
    g = graph_of(hanf, case["graph"])
    eng = port.engine(g.num_nodes(), g.offsets(), g.arcs(), **case["cfg"])
    assert float.hex(eng.sum_estimates()) == case["sum0"]
    assert sha(eng.counters()) == case["counters0_sha256"]
    for step in case["steps"]:
        s, m = eng.step()
        assert (float.hex(s), m) == (step["sum"], step["modified"]), (case["name"], step["t"])
        assert sha(eng.counters()) == step["counters_sha256"], (case["name"], step["t"])
        assert eng.systolic_active() == step["systolic"], (case["name"], step["t"])
    eng2 = port.engine(g.num_nodes(), g.offsets(), g.arcs(), **case["cfg"])
    vals, mods = eng2.run()
    assert [float.hex(v) for v in vals] == case["run_values"]
    assert mods == case["run_modified"]
    if "stats" in case:
        mean, var, spid = port.distance_distribution(vals)
        st = case["stats"]
        assert (float.hex(mean), float.hex(var), float.hex(spid)) == \
            (st["mean"], st["variance"], st["spid"])
        assert float.hex(port.effective_diameter(vals, 0.9, False)) == st["ed"]
        assert float.hex(port.effective_diameter(vals, 0.9, True)) == st["ied"]


def test_port_primitives_match_reference(port, primitives):
    """counter_estimate (hll.hpp:122-141) and PackedMax / naive union
    (broadword.hpp:94-130, hll.hpp:144-156) on random counters."""
    for lay in primitives:
        p = port.params(lay["b"], 0, lay["r"])
        for c in lay["cases"]:
            x = np.array(c["x"], dtype=np.uint64)
            y = np.array(c["y"], dtype=np.uint64)
            assert float.hex(port.estimate(x, p)) == c["estimate_x"]
            u = x.copy()
            assert bool(port.packed_max_into(p, u, y)) == c["changed"]
            assert [int(v) for v in u] == c["union"]
            n = x.copy()
            assert bool(port.naive_union(n, y, p)) == c["changed"]
            assert [int(v) for v in n] == c["union"]


def test_exhaustive_straddling_union(port):
    """test_hll.cpp:145-169: 2^20 value pairs of the straddling registers 12/13."""
    assert port.L.or_selftest_straddle() == 0


def test_estimate_known_answers(port):
    """test_hll.cpp:86-106: all-zero -> 0; all-ones m=16 -> 0.673*256/8;
    a single item -> m*ln(m/(m-1)) for every supported m."""
    p = port.params(4, 0)
    c = np.zeros(p.words, dtype=np.uint64)
    assert port.estimate(c, p) == 0.0
    for j in range(16):
        port.write_register(c, p, j, 1)
    assert port.estimate(c, p) == pytest.approx(0.673 * 256.0 / 8.0)
    for b in range(4, 15):
        p = port.params(b, 5)
        c = port.counter_of(p, [7777])
        m = float(1 << b)
        assert port.estimate(c, p) == pytest.approx(m * math.log(m / (m - 1.0)))


def test_clique_path_known_answer(port, recorded):
    """acceptance.cpp:252-263 / test_output.txt:14: T = 11, final jump 71722.3."""
    n, off, succ = port.gen_clique_path(260, 10)
    vals, _ = port.engine(n, off, succ, bucket_bits=8, seed=42).run()
    rec = recorded["clique_path_260_10"]
    assert len(vals) - 1 == rec["T"]
    assert f"{vals[-1] - vals[-2]:.6g}" == rec["final_jump"]


def test_exact_nf_closed_form(port):
    """acceptance.cpp:287-313: BFS == closed form on the (k<=8, l<=6) grid."""
    for k in range(1, 9):
        for l in range(1, 7):
            n, off, succ = port.gen_clique_path(k, l)
            nf = port.exact_nf(n, off, succ)
            assert nf == [port.clique_path_nf(k, l, t) for t in range(len(nf))]


def test_ball_counters(port):
    """test_engine.cpp:86-107: after t iterations counter v equals the
    counter fed B(v, t)."""
    n, off, succ = port.gen_uniform_random(60, 3, 21)
    for r in (5, 6):
        p = port.params(6, 77, r)
        eng = port.engine(n, off, succ, bucket_bits=6, register_bits=r, seed=77)
        for t in range(1, 5):
            eng.step()
            c = eng.counters().reshape(n, p.words)
            for v in range(n):
                assert np.array_equal(c[v], port.counter_of_ball(n, off, succ, v, t, p))


def test_port_vs_reference_live(ref, port, hanf):
    """The restatement against the reference engine itself, random configs
    including the optimisation toggles (test_engine.cpp:162-184)."""
    rng = np.random.default_rng(7)
    for trial in range(12):
        n = int(rng.integers(2, 400))
        d = int(rng.integers(0, min(n - 1, 9) + 1))
        seed = int(rng.integers(0, 1 << 40))
        g = hanf.gen_uniform_random(n, d, int(rng.integers(0, 1000)))
        cfg = dict(bucket_bits=int(rng.integers(4, 10)), register_bits=int(rng.choice([0, 5, 6, 7, 8])),
                   seed=seed, track_modified=bool(trial % 2), use_systolic=bool(trial % 3),
                   systolic_threshold=float(rng.choice([0.25, 1.0, 0.5])))
        rg = ref.graph(n, g.offsets(), g.arcs())
        re = ref.engine(rg, **cfg)
        pe = port.engine(n, g.offsets(), g.arcs(), **cfg)
        assert re.sum_estimates() == pe.sum_estimates()
        for _ in range(n + 1):
            a, b = re.step(), pe.step()
            assert a == b
            assert np.array_equal(re.counters(), pe.counters())
            if a[1] == 0:
                break


def test_recorded_unbiasedness_m64(port, recorded):
    """acceptance.cpp:204-228 / test_output.txt:11 (worst |mean/exact - 1| =
    0.01486 over 100 seeds at m = 64): reproduced digit for digit."""
    n, off, succ = port.gen_uniform_random(1000, 8, 4242)
    exact = port.exact_nf(n, off, succ)
    L = len(exact)
    mean = np.zeros(L)
    for i in range(100):
        vals, _ = port.engine(n, off, succ, bucket_bits=6, seed=100 + i).run()
        mean += [vals[t] if t < len(vals) else vals[-1] for t in range(L)]
    mean /= 100
    worst = max(abs(mean[t] / exact[t] - 1.0) for t in range(L))
    assert f"{worst:.4g}" == recorded["unbiasedness_m64_worst"]["value"]
