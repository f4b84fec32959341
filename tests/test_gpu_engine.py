"""Parity of the B200 engine (libhanf.so through its C-ABI) with the
reference: golden traces made by the reference engine, the CPU oracle run
in lockstep, the reference's own known answers and recorded acceptance
values, and size-independent properties at BASELINE config 2 scale."""
from __future__ import annotations

import hashlib
import math
import os

import numpy as np
import pytest

from conftest import graph_of

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def lockstep(hanf, port, g, max_steps=None, exact=True, **cfg):
    """GPU engine vs oracle after every iteration: counters bit-exact,
    modified exact, N(t) bit-exact (exact_sum) or within 1e-12 relative."""
    pe = port.engine(g.num_nodes(), g.offsets(), g.arcs(),
                     **{k: v for k, v in cfg.items() if k in
                        ("bucket_bits", "register_bits", "seed", "systolic_threshold",
                         "track_modified", "use_systolic")})
    with hanf.NfEngine(g, hanf.EngineConfig(exact_sum=exact, **cfg)) as e:
        assert np.array_equal(e.counters(), pe.counters())
        s0 = pe.sum_estimates()
        assert e.sum_estimates() == s0 if exact else math.isclose(e.sum_estimates(), s0, rel_tol=1e-12)
        steps = 0
        while True:
            r = e.step()
            s, m = pe.step()
            steps += 1
            assert r.modified == m, steps
            if exact:
                assert r.sum == s, steps
            else:
                assert math.isclose(r.sum, s, rel_tol=1e-12), steps
            assert np.array_equal(e.counters(), pe.counters()), steps
            assert e.systolic_active() == pe.systolic_active()
            assert e.iteration() == pe.iteration()
            if m == 0 or (max_steps and steps >= max_steps):
                return steps


@pytest.mark.parametrize("idx", range(28))
def test_golden_trace(hanf, traces, idx):
    """Every iteration of the reference engine's trace, reproduced."""
    if idx >= len(traces):
        pytest.skip("fewer golden cases")
    case = traces[idx]
    g = graph_of(hanf, case["graph"])
    with hanf.NfEngine(g, hanf.EngineConfig(**case["cfg"])) as e:
        assert float.hex(e.sum_estimates()) == case["sum0"]
        assert sha(e.counters()) == case["counters0_sha256"]
        if "counters0" in case:
            assert [int(x) for x in e.counters()] == case["counters0"]
        for step in case["steps"]:
            r = e.step()
            assert (float.hex(r.sum), r.modified) == (step["sum"], step["modified"]), step["t"]
            assert sha(e.counters()) == step["counters_sha256"], step["t"]
            assert e.systolic_active() == step["systolic"]
        e.reset()
        est = e.run_to_stabilisation()
        assert [float.hex(v) for v in est.values] == case["run_values"]
        assert est.modified == case["run_modified"]
    if "stats" in case:
        d = hanf.distance_distribution(est.values)
        st = case["stats"]
        assert (float.hex(d.mean), float.hex(d.variance), float.hex(d.spid)) == \
            (st["mean"], st["variance"], st["spid"])
        assert float.hex(hanf.effective_diameter(est.values, 0.9, False)) == st["ed"]
        assert float.hex(hanf.effective_diameter(est.values, 0.9, True)) == st["ied"]


def test_lockstep_knobs_and_layouts(hanf, port):
    """Optimisation toggles change time only, never bits (test_engine.cpp:162-184);
    every register width and counter size the kernels specialise."""
    rng = np.random.default_rng(11)
    graphs = [hanf.gen_uniform_random(3000, 6, 2), hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 3, 5),
              hanf.gen_clique_path(40, 7), hanf.Graph.from_edges(5, [(0, 1), (1, 2), (2, 0)])]
    for g in graphs:
        for b, r in [(4, 5), (5, 5), (6, 5), (7, 5), (8, 5), (9, 5), (6, 6), (6, 7), (5, 8)]:
            knobs = dict(track_modified=bool(rng.integers(2)), use_systolic=bool(rng.integers(2)),
                         systolic_threshold=float(rng.choice([0.25, 1.0])))
            lockstep(hanf, port, g, bucket_bits=b, register_bits=r,
                     seed=int(rng.integers(1 << 62)), **knobs)


def test_device_sum_mode(hanf, port):
    """exact_sum = False: deterministic device tree; within 1e-12 relative
    (north_star bound 1e-9), counters unaffected."""
    g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 1, 7)
    lockstep(hanf, port, g, exact=False, bucket_bits=6, seed=42)
    a = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=42, exact_sum=False))
    b = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=42, exact_sum=False))
    assert a.values == b.values  # reruns bit-identical


def test_balls(hanf, port):
    """test_engine.cpp:86-107: counter v after t iterations == counter of B(v, t)."""
    g = hanf.gen_uniform_random(60, 3, 21)
    for r in (5, 6):
        p = port.params(6, 77, r)
        with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, register_bits=r, seed=77)) as e:
            for t in range(1, 5):
                e.step()
                c = e.counters().reshape(60, p.words)
                for v in range(60):
                    ball = port.counter_of_ball(60, g.offsets(), g.arcs(), v, t, p)
                    assert np.array_equal(c[v], ball), (r, t, v)


def test_single_arc_and_three_path(hanf, port):
    """test_engine.cpp:63-83 (rep.sum == exact sum of the two estimates) and
    :109-133 (N(t) = sums of ball-fed counters)."""
    g = hanf.Graph.from_edges(2, [(0, 1)])
    p = port.params(7, 9)
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=7, seed=9)) as e:
        rep = e.step()
        both = port.counter_of(p, [0, 1])
        just1 = port.counter_of(p, [1])
        assert np.array_equal(e.counter(0), both) and np.array_equal(e.counter(1), just1)
        assert rep.modified <= 1
        assert rep.sum == port.estimate(both, p) + port.estimate(just1, p)
        assert rep.sum == pytest.approx(3.0, abs=0.3)
    g3 = hanf.Graph.from_edges(3, [(0, 1), (1, 2)])
    p = port.params(7, 5)
    est = hanf.estimate_nf(g3, hanf.EngineConfig(bucket_bits=7, seed=5))
    assert len(est.values) == 3 and est.modified[0] == 3
    for t in range(3):
        s = 0.0
        for v in range(3):
            s += port.estimate(port.counter_of_ball(3, g3.offsets(), g3.arcs(), v, t, p), p)
        assert est.values[t] == s


def test_edge_cases(hanf):
    """Empty graph, arcless graph, isolated nodes, iteration cap, bad index."""
    empty = hanf.Graph.from_edges(0, [])
    est = hanf.estimate_nf(empty, hanf.EngineConfig())
    assert est.values == [] and est.iterations() == 0
    with hanf.NfEngine(empty, hanf.EngineConfig()) as e:
        assert e.step().modified == 0
    arcless = hanf.Graph.from_edges(5, [])
    with hanf.NfEngine(arcless, hanf.EngineConfig(bucket_bits=7, seed=1)) as e:
        before = e.sum_estimates()
        rep = e.step()
        assert rep.modified == 0 and rep.sum == before
        with pytest.raises(IndexError):
            e.counter(5)
        with pytest.raises(IndexError):
            e.counters(3, 4)
    single = hanf.Graph.from_edges(1, [])
    with hanf.NfEngine(single, hanf.EngineConfig(bucket_bits=7, seed=3)) as e:
        assert 0.9 < e.sum_estimates() < 1.1
    cap = hanf.gen_clique_path(4, 8)
    with pytest.raises(hanf.GuardError, match="iteration cap 2"):
        hanf.estimate_nf(cap, hanf.EngineConfig(bucket_bits=6, seed=1, max_iterations=2))
    loops = hanf.Graph.from_edges(3, [(0, 0), (1, 1), (1, 2)])
    est = hanf.estimate_nf(loops, hanf.EngineConfig(bucket_bits=6, seed=2))
    assert est.modified[0] == 3


def test_reruns_reset_and_seeds(hanf):
    """test_engine.cpp:135-143: same seed -> same values; other seed differs."""
    g = hanf.gen_uniform_random(400, 6, 13)
    a = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=99))
    b = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=99))
    c = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=100))
    assert a.values == b.values and a.modified == b.modified and a.values != c.values
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=99)) as e:
        first = e.run_to_stabilisation()
        e.reset()
        assert e.iteration() == 0
        assert e.run_to_stabilisation().values == first.values == a.values


def test_threshold_termination(hanf):
    """test_engine.cpp:228-245: eps_inc 0.01 stops inside the plateau and
    misses the final k^2 jump; stabilisation reaches T = 11."""
    g = hanf.gen_clique_path(260, 10)
    full = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=7, seed=6))
    assert full.iterations() == 11
    trunc = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=7, seed=6,
                                                  termination=hanf.Termination.threshold,
                                                  eps_inc=0.01))
    assert trunc.iterations() < full.iterations()
    assert full.values[-1] - trunc.values[-1] > 0.5 * 260 * 260
    assert hanf.effective_diameter(trunc.values, 0.9) == 1.0


def test_systolic_activation(hanf):
    """test_engine.cpp:186-205 on the 64-path."""
    g = hanf.Graph.from_edges(64, [(v, v + 1) for v in range(63)])
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=2)) as e:
        steps = 0
        while e.step().modified > 0:
            steps += 1
        assert e.systolic_active() and steps >= 32
    off = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=2, use_systolic=False))
    assert len(off.values) == steps + 1 <= 64


def test_recorded_clique_path(hanf, recorded):
    """test_output.txt:14: T = 11, final jump 71722.3 (b = 8, seed 42)."""
    est = hanf.estimate_nf(hanf.gen_clique_path(260, 10), hanf.EngineConfig(bucket_bits=8, seed=42))
    rec = recorded["clique_path_260_10"]
    assert est.iterations() == rec["T"]
    assert f"{est.values[-1] - est.values[-2]:.6g}" == rec["final_jump"]


def _unbiasedness(hanf, port, b):
    g = hanf.gen_uniform_random(1000, 8, 4242)
    exact = port.exact_nf(1000, g.offsets(), g.arcs())
    L = len(exact)
    mean = np.zeros(L)
    for i in range(100):
        v = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=b, seed=100 + i)).values
        mean += [v[t] if t < len(v) else v[-1] for t in range(L)]
    mean /= 100
    return max(abs(mean[t] / exact[t] - 1.0) for t in range(L))


def test_recorded_unbiasedness(hanf, port, recorded):
    """test_output.txt:11-12 (acceptance criteria 4 / 4x): worst deviation of
    the 100-seed mean, m = 64 and m = 1024, digit for digit."""
    assert f"{_unbiasedness(hanf, port, 6):.4g}" == recorded["unbiasedness_m64_worst"]["value"]
    assert f"{_unbiasedness(hanf, port, 10):.4g}" == recorded["unbiasedness_m1024_worst"]["value"]


def test_recorded_concentration(hanf, port, recorded):
    """test_output.txt:13 (criterion 5): 97/100 within 2 eta, 100/100 within 3."""
    g = hanf.gen_uniform_random(1000, 8, 4242)
    exact = port.exact_nf(1000, g.offsets(), g.arcs())
    eta = 1.06 / 16.0
    w2 = w3 = 0
    for i in range(100):
        v = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=8, seed=300 + i)).values
        worst = max(abs((v[t] if t < len(v) else v[-1]) / exact[t] - 1.0) for t in range(len(exact)))
        w2 += worst <= 2 * eta
        w3 += worst <= 3 * eta
    rec = recorded["concentration_m256"]
    assert (w2, w3) == (rec["within2"], rec["within3"])


def test_recorded_spid(hanf, port, recorded):
    """test_output.txt:23 (criterion 9): multirun spid means and relative sd."""
    web = hanf.gen_clique_path(252, 10)
    social = hanf.gen_uniform_random(1000, 20, 2020)
    exact = [hanf.distance_distribution(port.exact_nf(g.num_nodes(), g.offsets(), g.arcs())).spid
             for g in (web, social)]
    rec = recorded["spid"]
    assert [f"{exact[0]:.3g}", f"{exact[1]:.3g}"] == rec["exact"]
    for rep, want in enumerate(rec["reps"]):
        base = 500 + rep * 1000
        got = []
        for g in (web, social):
            runs = [hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=7, seed=base + i))
                    for i in range(100)]
            agg = hanf.aggregate_runs(runs)
            got += [f"{agg.mean.spid:.3g}", f"{agg.stddev.spid / agg.mean.spid:.2g}"]
        assert got == want, rep


def test_config2_scale(hanf, port):
    """BASELINE config 2 (R-MAT scale 20, 16.1 M arcs): lockstep against the
    reference engine for every iteration when it is available, and
    size-independent properties: non-decreasing N(t), stabilised counters are
    a fixed point, sampled counters equal the counters of their balls."""
    import oracle
    g = hanf.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7)
    n = g.num_nodes()
    cfg = dict(bucket_bits=6, seed=42)
    p = port.params(6, 42)
    with hanf.NfEngine(g, hanf.EngineConfig(**cfg)) as e:
        if oracle.have_ref():
            ref = oracle.ref()
            re = ref.engine(ref.graph(n, g.offsets(), g.arcs()), threads=os.cpu_count() or 1, **cfg)
            assert e.sum_estimates() == re.sum_estimates()
            while True:
                r = e.step()
                s, m = re.step()
                assert (r.sum, r.modified) == (s, m)
                assert np.array_equal(e.counters(), re.counters())
                if m == 0:
                    break
            e.reset()
        est = e.run_to_stabilisation()
        assert all(b >= a for a, b in zip(est.values, est.values[1:]))
        final = e.counters().reshape(n, p.words)
        T = est.iterations()
        assert e.step().modified == 0
        rng = np.random.default_rng(1)
        for v in rng.choice(n, 12, replace=False):
            ball = port.counter_of_ball(n, g.offsets(), g.arcs(), int(v), T + 1, p)
            assert np.array_equal(final[v], ball), v


@pytest.mark.parametrize("b,env,delta", [(6, {}, False), (6, {"HANF_SPARSE": "1"}, False),
                                         (5, {}, False), (8, {}, False), (6, {}, True),
                                         (5, {"HANF_SPARSE": "1"}, True), (8, {}, True),
                                         (6, {"HANF_SEGMENTS": "1"}, True),
                                         (7, {"HANF_SEGMENTS": "1", "HANF_SUMMARY": "1"}, False)])
def test_sharded_engines_exchange(hanf, port, monkeypatch, b, env, delta):
    """The shard ABI (hanf_shard_compute / device buffers / hanf_shard_commit)
    on one GPU: two node-range engines, exchange done by device copies in
    sequence (no kernel waits on another), equal to one engine bit for bit;
    with the worklist step, the padded W = 3 rows and a multi-chunk layout."""
    import torch
    from paper_1011_5599_b200.sharded import LocalCudaShard, shard_ranges
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    g = hanf.gen_rmat(14, 16, 0.57, 0.19, 0.19, 1, 7)
    n = g.num_nodes()
    cfg = hanf.EngineConfig(bucket_bits=b, seed=42)
    dev = torch.device("cuda", 0)
    shards = [LocalCudaShard(g, cfg, lo, hi, dev) for lo, hi in shard_ranges(n, 2)]
    ranges = shard_ranges(n, 2)
    values = [shards[0].sum_estimates()]
    mods = [n]
    words = shards[0].row_words()
    packets = [(torch.empty(n, dtype=torch.int32, device=dev),
                torch.empty(n * words, dtype=torch.int64, device=dev)) for _ in shards]
    rows_steps = 0
    while True:
        for sh in shards:
            sh.shard_compute()
        torch.cuda.synchronize()
        # changed-rows exchange from the second step on (hanf_shard_pack/unpack)
        use_rows = delta and len(values) > 1
        if use_rows:
            counts = [sh.pack_rows(*packets[k]) for k, sh in enumerate(shards)]
            for k in range(2):
                shards[1 - k].unpack_rows(packets[k][0], packets[k][1], counts[k])
            rows_steps += 1
        bufs = [sh.exchange_buffers() for sh in shards]
        for k, (lo, hi) in enumerate(ranges):
            for b_idx, (t_own, unit, per_node) in enumerate(bufs[k]):
                if per_node is not None and use_rows:
                    continue
                span = (lo * per_node, hi * per_node) if per_node else (lo // 64, -(-hi // 64))
                for j in range(2):
                    if j != k:
                        bufs[j][b_idx][0][span[0]:span[1]].copy_(t_own[span[0]:span[1]])
        torch.cuda.synchronize()
        reps = [sh.shard_commit() for sh in shards]
        assert reps[0].sum == reps[1].sum and reps[0].modified == reps[1].modified
        if reps[0].modified == 0:
            break
        values.append(reps[0].sum)
        mods.append(reps[0].modified)
    single = hanf.estimate_nf(g, cfg)
    assert values == single.values and mods == single.modified
    assert (rows_steps > 0) == delta
    a = shards[0].engine.counters()
    assert np.array_equal(a, shards[1].engine.counters())
    with hanf.NfEngine(g, cfg) as e:
        e.run_to_stabilisation()
        assert np.array_equal(a, e.counters())
    for sh in shards:
        sh.close()


def test_launch_accounting(hanf):
    g = hanf.gen_uniform_random(5000, 8, 1)
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=1)) as e:
        before = e.launch_count()
        e.step()
        assert e.launch_count() - before >= 2  # union sweep + finish


def test_worklist_step_parity(hanf, port, monkeypatch):
    """The worklist step (engine.hpp:210-224 systolic mode; on by default
    below n/128 changed counters on graphs from 2^22 arcs, forced here with
    HANF_SPARSE=1) changes time only: lockstep bit-exact with the oracle."""
    monkeypatch.setenv("HANF_SPARSE", "1")
    for g in (hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 2, 3),
              hanf.Graph.from_edges(300, [(v, v + 1) for v in range(299)]),
              hanf.gen_clique_path(30, 40)):
        for b in (5, 6, 7):
            lockstep(hanf, port, g, bucket_bits=b, seed=9)


@pytest.mark.parametrize("env", [{}, {"HANF_RELABEL": "1"}, {"HANF_RELABEL": "1", "HANF_SPARSE": "1"},
                                 {"HANF_SUMMARY": "1"}, {"HANF_SUMMARY": "1", "HANF_RELABEL": "1"},
                                 {"HANF_SEGMENTS": "1"}, {"HANF_SEGMENTS": "1", "HANF_SUMMARY": "1"},
                                 {"HANF_SEGMENTS": "1", "HANF_SPARSE": "1"}])
def test_row_pitch_and_gather_variants(hanf, port, monkeypatch, env):
    """Every layout's gather (padded W = 3 rows with aligned 256-bit loads,
    16-byte windows, per-word loads, multi-chunk counters) under each
    schedule change time only: counters read back in the reference packing
    and bit-exact in lockstep with the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for g in (hanf.gen_rmat(11, 16, 0.57, 0.19, 0.19, 4, 6), hanf.gen_clique_path(20, 9)):
        for b, r in [(4, 5), (5, 5), (6, 5), (7, 5), (5, 6), (5, 7), (6, 7)]:
            lockstep(hanf, port, g, bucket_bits=b, register_bits=r, seed=77)


def test_pinned_graph_upload(hanf):
    """Graph.pin() (hanf_pin_host) changes the upload path only."""
    g = hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 5, 9)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=3)
    a = hanf.estimate_nf(g, cfg)
    p = hanf.Graph(g.num_nodes(), g.offsets().copy(), g.arcs().copy()).pin()
    b = hanf.estimate_nf(p, cfg)
    p.unpin()
    p.unpin()  # idempotent
    assert list(a.values) == list(b.values) and list(a.modified) == list(b.modified)
    with pytest.raises(Exception):
        hanf._lib.check(hanf._lib.lib().hanf_pin_host(None, 8))


@pytest.mark.parametrize("idx", range(28))
def test_golden_trace_relabelled(hanf, traces, idx, monkeypatch):
    """Degree relabelling is an internal layout: every golden iteration,
    counter read-back and N(t) bit is unchanged (HANF_RELABEL=1 forces it
    on graphs the default heuristic leaves alone)."""
    monkeypatch.setenv("HANF_RELABEL", "1")
    test_golden_trace(hanf, traces, idx)


@pytest.mark.parametrize("idx", range(28))
def test_golden_trace_segmented(hanf, traces, idx, monkeypatch):
    """Segmented tasks (light tasks grouped by node segment; skip sweeps drop
    the segments with no modified row in reach) change time only: every
    golden iteration bit-exact (HANF_SEGMENTS=1 forces them on)."""
    monkeypatch.setenv("HANF_SEGMENTS", "1")
    test_golden_trace(hanf, traces, idx)


@pytest.mark.parametrize("env", [{}, {"HANF_SEGMENTS": "1"}])
def test_create_lockstep_and_reset(hanf, port, monkeypatch, env):
    """Lockstep with the oracle, then reset / reseed re-run every step in
    full, and bad arcs are rejected at create."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 2, 3)
    for b in (5, 6, 7):
        lockstep(hanf, port, g, bucket_bits=b, seed=21)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=21)
    ref = hanf.estimate_nf(g, cfg)
    with hanf.NfEngine(g, cfg) as e:
        e.step()
        e.reset()
        assert e.run_to_stabilisation().values == ref.values
        e.reseed(22)
        other = e.run_to_stabilisation()
    assert other.values == hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=22)).values
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    arcs = g.arcs().copy()
    arcs[len(arcs) // 2] = g.num_nodes() + 5
    bad = hanf.Graph(g.num_nodes(), g.offsets().copy(), arcs)
    with pytest.raises(ValueError):
        hanf.NfEngine(bad, cfg)
    with hanf.NfEngine(g, cfg) as e:  # the device is fine afterwards
        assert e.run_to_stabilisation().values == ref.values


@pytest.mark.parametrize("env", [{}, {"HANF_SPARSE": "0"}, {"HANF_SUMMARY": "1"}])
def test_segmented_copying_graph(hanf, port, monkeypatch, env):
    """A config-3-shaped copying graph (local ids: segmented by default from
    2^20 nodes, forced here at 2^15) run to stabilisation in lockstep with
    the oracle: the long tail of skip sweeps visits a few segments only."""
    monkeypatch.setenv("HANF_SEGMENTS", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = hanf.gen_copying(1 << 15, 2.1, 8.0, 300, 0.6, 64, 3)
    lockstep(hanf, port, g, bucket_bits=5, seed=42)


def test_relabel_multichunk_and_readback(hanf, port, monkeypatch):
    """Relabelled multi-chunk layouts (separate estimate kernel over
    original-id blocks) and partial counter read-back ranges."""
    monkeypatch.setenv("HANF_RELABEL", "1")
    g = hanf.gen_rmat(11, 8, 0.57, 0.19, 0.19, 8, 1)
    for b, r in [(8, 5), (9, 5), (7, 6), (8, 7), (6, 8)]:
        lockstep(hanf, port, g, bucket_bits=b, register_bits=r, seed=5, max_steps=4)
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=5)) as e:
        e.step()
        full = e.counters()
        W = e.params().words
        for first, count in [(0, 1), (17, 33), (g.num_nodes() - 5, 5)]:
            part = e.counters(first, count)
            assert np.array_equal(part, full[first * W:(first + count) * W])


def test_multirun_reseed(hanf):
    """multirun (main.cpp:263-283): one engine re-seeded per run gives each
    seed's estimate_nf bit for bit; aggregate_runs takes the list."""
    g = hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 2, 4)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=100)
    runs = hanf.multirun(g, cfg, runs=4)
    assert cfg.seed == 100  # caller's config untouched
    for i, r in enumerate(runs):
        ref = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=100 + i))
        assert r.values == ref.values and r.modified == ref.modified and r.seed == 100 + i
    rep = hanf.aggregate_runs(runs)
    assert rep is not None


def test_hca1_snapshot_and_resume(hanf, ref, tmp_path, monkeypatch):
    """HCA1 snapshots (hll.hpp:241-305): the engine's file is byte for byte
    the reference's save_counters output after the same iterations, and an
    engine restored from it continues exactly like the uninterrupted run."""
    g = hanf.gen_rmat(11, 16, 0.57, 0.19, 0.19, 6, 2)
    for relabel in ("0", "1"):
        monkeypatch.setenv("HANF_RELABEL", relabel)
        for b, r in [(6, 5), (5, 5), (8, 5), (6, 7)]:
            re = ref.engine(ref.graph(g.num_nodes(), g.offsets(), g.arcs()), bucket_bits=b,
                            register_bits=r, seed=11)
            cfg = hanf.EngineConfig(bucket_bits=b, register_bits=r, seed=11)
            with hanf.NfEngine(g, cfg) as e:
                for _ in range(2):
                    e.step()
                    re.step()
                ours, theirs = tmp_path / "ours.hca", tmp_path / "ref.hca"
                e.save_counters(ours)
                re.save_counters(theirs)
                assert ours.read_bytes() == theirs.read_bytes()
                at2 = e.sum_estimates()
                rest = []
                while True:  # the uninterrupted run from iteration 3 on
                    rep = e.step()
                    rest.append((rep.sum, rep.modified, e.counters()))
                    if rep.modified == 0:
                        break
            with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=b, register_bits=r, seed=99)) as e:
                e.restore_counters(ours, iteration=2)
                assert e.iteration() == 2 and e.params().seed == 11
                assert e.sum_estimates() == at2
                for s_, m_, c_ in rest:
                    rep = e.step()
                    assert (rep.sum, rep.modified) == (s_, m_)
                    assert np.array_equal(e.counters(), c_)
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=7, seed=11)) as e:
        with pytest.raises(ValueError):
            e.restore_counters(ours)  # b mismatch
        bad = tmp_path / "bad.hca"
        bad.write_bytes(b"XXXX" + bytes(40))
        with pytest.raises(Exception):
            e.restore_counters(bad)


@pytest.mark.parametrize("batch", [2, 4, 8])
def test_batched_runs_equal_single_runs(hanf, monkeypatch, batch):
    """Batched runs (hanf_create_batch: the graph lifted to K copies) give
    every seed's estimate_nf bit for bit, over layouts, the worklist step and
    a multi-chunk layout."""
    for sparse in ("0", "1"):
        monkeypatch.setenv("HANF_SPARSE", sparse)
        for g, b, r in [(hanf.gen_rmat(11, 16, 0.57, 0.19, 0.19, 3, 8), 6, 5),
                        (hanf.gen_clique_path(12, 30), 5, 5),
                        (hanf.gen_uniform_random(1500, 3, 4), 8, 5),
                        (hanf.gen_rmat(10, 8, 0.57, 0.19, 0.19, 5, 1), 5, 7)]:
            cfg = hanf.EngineConfig(bucket_bits=b, register_bits=r, seed=1000)
            runs = hanf.multirun(g, cfg, runs=batch + 1, batch=batch)
            for i, est in enumerate(runs):
                ref = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=b, register_bits=r,
                                                            seed=1000 + i))
                assert est.values == ref.values and est.modified == ref.modified, (i, b, r)


def test_batched_engine_rejects_single_run_calls(hanf):
    import ctypes
    from ctypes import c_uint64, c_void_p
    g = hanf.gen_uniform_random(100, 2, 1)
    view, cfg = g.view(), hanf.EngineConfig(bucket_bits=5).to_c()
    seeds = (c_uint64 * 3)(1, 2, 3)
    h = c_void_p()
    assert hanf._lib.lib().hanf_create_batch(ctypes.byref(view), ctypes.byref(cfg), seeds, 3,
                                             ctypes.byref(h)) != 0  # runs must be 2, 4, 8
    seeds = (c_uint64 * 2)(1, 2)
    hanf._lib.check(hanf._lib.lib().hanf_create_batch(ctypes.byref(view), ctypes.byref(cfg),
                                                      seeds, 2, ctypes.byref(h)))
    rep = hanf._lib.IterationReportC()
    assert hanf._lib.lib().hanf_step(h, ctypes.byref(rep)) != 0
    hanf._lib.lib().hanf_destroy(h)


def test_step_launch_complete(hanf):
    """hanf_step_launch / hanf_step_complete = hanf_step, split at the device
    boundary; misuse is an invalid argument."""
    g = hanf.gen_rmat(11, 16, 0.57, 0.19, 0.19, 1, 2)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=9)
    with hanf.NfEngine(g, cfg) as a, hanf.NfEngine(g, cfg) as b:
        while True:
            ra = a.step()
            b.step_launch()
            with pytest.raises(ValueError):
                b.step()  # a launched step is pending
            rb = b.step_complete()
            assert (ra.sum, ra.modified) == (rb.sum, rb.modified)
            assert np.array_equal(a.counters(), b.counters())
            if ra.modified == 0:
                break
        with pytest.raises(ValueError):
            b.step_complete()


@pytest.mark.parametrize("layout", ["packed", "bytes"])
def test_golden_traces_each_counter_layout(hanf, traces, monkeypatch, layout):
    """Both device counter stores (byte registers, the default for
    L2-resident arrays, and the reference packing) reproduce every golden
    trace bit for bit: the layout changes time only."""
    monkeypatch.setenv("HANF_LAYOUT", layout)
    for case in traces:
        g = graph_of(hanf, case["graph"])
        with hanf.NfEngine(g, hanf.EngineConfig(**case["cfg"])) as e:
            assert sha(e.counters()) == case["counters0_sha256"]
            for step in case["steps"]:
                r = e.step()
                assert (float.hex(r.sum), r.modified) == (step["sum"], step["modified"]), step["t"]
                assert sha(e.counters()) == step["counters_sha256"], step["t"]
            e.reset()
            est = e.run_to_stabilisation()
            assert [float.hex(v) for v in est.values] == case["run_values"]


@pytest.mark.parametrize("env", [{"HANF_LAYOUT": "bytes", "HANF_RELABEL": "1"},
                                 {"HANF_LAYOUT": "bytes", "HANF_SPARSE": "1"},
                                 {"HANF_LAYOUT": "bytes", "HANF_SEGMENTS": "1", "HANF_SUMMARY": "1"},
                                 {"HANF_LAYOUT": "bytes", "HANF_RELABEL": "1", "HANF_SPARSE": "1"},
                                 {"HANF_LAYOUT": "packed", "HANF_SPARSE": "1"}])
def test_byte_layout_paths(hanf, port, monkeypatch, env):
    """Byte-layout rows through every path that touches them: relabelled
    rows, the worklist step, segmented skip sweeps with the summary probe,
    hub chunks (clique-path hubs) and m = 16..128; lockstep with the
    oracle, counters read back in the reference packing."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for g in (hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 3, 5), hanf.gen_clique_path(1500, 3)):
        for b in (4, 5, 6, 7):
            lockstep(hanf, port, g, bucket_bits=b, seed=1234 + b)


def test_byte_layout_snapshot_restore(hanf, monkeypatch, tmp_path):
    """HCA1 snapshots written from byte rows are the reference packing, and
    restoring them into either layout resumes bit for bit."""
    g = hanf.gen_rmat(11, 8, 0.57, 0.19, 0.19, 2, 9)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=5)
    monkeypatch.setenv("HANF_LAYOUT", "packed")
    with hanf.NfEngine(g, cfg) as ref:
        ref.step(), ref.step()
        want = ref.counters()
        ref.save_counters(str(tmp_path / "p.hca"))
    monkeypatch.setenv("HANF_LAYOUT", "bytes")
    with hanf.NfEngine(g, cfg) as e:
        e.step(), e.step()
        assert np.array_equal(e.counters(), want)
        e.save_counters(str(tmp_path / "b.hca"))
        assert (tmp_path / "b.hca").read_bytes() == (tmp_path / "p.hca").read_bytes()
        e.reset()
        e.restore_counters(str(tmp_path / "p.hca"))
        assert np.array_equal(e.counters(), want)


@pytest.mark.parametrize("env", [{"HANF_TASKSCAN": "1"},
                                 {"HANF_TASKSCAN": "1", "HANF_LAYOUT": "packed"},
                                 {"HANF_TASKSCAN": "1", "HANF_RELABEL": "1"},
                                 {"HANF_TASKSCAN": "1", "HANF_RELABEL": "1", "HANF_LAYOUT": "packed"}])
def test_task_scan_step(hanf, port, traces, monkeypatch, env):
    """Mode 4 (one flat TOS scan lists the tasks in reach of a change, the
    skip sweep runs on that list, stale rows outside it are copied) forced
    on every skip step: every golden trace and lockstep runs with hubs,
    relabelled rows and both counter stores stay bit-exact."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for case in traces:
        g = graph_of(hanf, case["graph"])
        with hanf.NfEngine(g, hanf.EngineConfig(**case["cfg"])) as e:
            for step in case["steps"]:
                r = e.step()
                assert (float.hex(r.sum), r.modified) == (step["sum"], step["modified"]), step["t"]
                assert sha(e.counters()) == step["counters_sha256"], step["t"]
            e.reset()
            est = e.run_to_stabilisation()
            assert [float.hex(v) for v in est.values] == case["run_values"]
    for g in (hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 3, 5), hanf.gen_clique_path(2000, 3),
              hanf.gen_uniform_random(5000, 3, 4)):
        lockstep(hanf, port, g, bucket_bits=6, seed=99)


@pytest.mark.parametrize("hot", ["0", "16", "1040"])
def test_relabel_line_slots(hanf, port, monkeypatch, hot):
    """Relabelled rows of an odd pitch past a hot prefix take line-aligned
    slots first (hanf_relabel.cu make_slots; on by default only past 2^22
    rows, forced small here): every counter read back, N(t) and the
    modified counts stay the reference's, for W = 5 and W = 7 rows."""
    monkeypatch.setenv("HANF_LAYOUT", "packed")
    monkeypatch.setenv("HANF_RELABEL", "1")
    monkeypatch.setenv("HANF_SLOTS_HOT", hot)
    for g in (hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 3, 5), hanf.gen_clique_path(700, 4),
              hanf.gen_uniform_random(3001, 4, 8)):
        lockstep(hanf, port, g, bucket_bits=6, seed=17)
        lockstep(hanf, port, g, bucket_bits=6, register_bits=7, seed=18)
