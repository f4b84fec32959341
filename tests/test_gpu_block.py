"""Source-blocked dense sweeps (hanf_block.cu): an engine-internal schedule
of NfEngine::step's union loop (engine.hpp:157-185) in which the arcs from
the rows of highest out-degree to the cold rows are folded one successor
segment at a time into extra item rows.  The reference's invariant is that
scheduling never changes a bit (test_engine.cpp:145-184): every counter, the
modified counts and N(t) must stay the oracle's and the golden traces'.
On by size only for config-5-like engines, so the shapes are forced small
here (HANF_BLOCK_S / _T / _SEG / _GROUP are log2 sizes)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import graph_of
from test_gpu_engine import lockstep, sha

pytestmark = pytest.mark.gpu

SHAPES = [
    # sources, cold rows from, rows per segment, items per task group
    {"HANF_BLOCK_S": "6", "HANF_BLOCK_T": "7", "HANF_BLOCK_SEG": "6", "HANF_BLOCK_GROUP": "6"},
    {"HANF_BLOCK_S": "10", "HANF_BLOCK_T": "4", "HANF_BLOCK_SEG": "8", "HANF_BLOCK_GROUP": "8"},
    {"HANF_BLOCK_S": "3", "HANF_BLOCK_T": "0", "HANF_BLOCK_SEG": "12", "HANF_BLOCK_GROUP": "18"},
]


def _force(monkeypatch, shape, mode="1"):
    monkeypatch.setenv("HANF_BLOCK", mode)
    monkeypatch.setenv("HANF_RELABEL", "1")
    monkeypatch.setenv("HANF_LAYOUT", "packed")
    for k, v in shape.items():
        monkeypatch.setenv(k, v)


def _graphs(hanf):
    return (hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 3, 5),  # hubs of > 1024 arcs
            hanf.gen_clique_path(1500, 3),                  # every clique node a hub
            hanf.gen_uniform_random(5000, 12, 4))


@pytest.mark.parametrize("shape", SHAPES)
def test_blocked_lockstep_with_oracle(hanf, port, monkeypatch, shape):
    _force(monkeypatch, shape)
    for g in _graphs(hanf):
        with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=5)) as e:
            items, arcs = e.block_stats()
            assert items > 0 and arcs >= items, (items, arcs)
        lockstep(hanf, port, g, bucket_bits=6, seed=99)
        lockstep(hanf, port, g, bucket_bits=6, register_bits=7, seed=98)
        lockstep(hanf, port, g, bucket_bits=5, seed=97, exact=False)


def test_blocked_golden_traces(hanf, traces, monkeypatch):
    _force(monkeypatch, SHAPES[0])
    used = 0
    for case in traces:
        g = graph_of(hanf, case["graph"])
        with hanf.NfEngine(g, hanf.EngineConfig(**case["cfg"])) as e:
            used += e.block_stats()[0] > 0
            for step in case["steps"]:
                r = e.step()
                assert (float.hex(r.sum), r.modified) == (step["sum"], step["modified"]), step["t"]
                assert sha(e.counters()) == step["counters_sha256"], step["t"]
            e.reset()
            est = e.run_to_stabilisation()
            assert [float.hex(v) for v in est.values] == case["run_values"]
    assert used > 0  # (graphs too small or too thin for items fall back to the plain sweep)


def test_blocked_from_the_first_reseed(hanf, monkeypatch):
    """HANF_BLOCK=2: the build at the first reset / reseed whatever the size
    (by default a large engine builds at the reset that follows its 96th
    dense step, tests/test_gpu_atsize.py).  The first run sweeps plainly,
    every later run equals a fresh engine's."""
    _force(monkeypatch, SHAPES[1], mode="2")
    g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 3, 5)
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=7)) as e:
        assert e.block_stats() == (0, 0)
        first = e.run_to_stabilisation()
        c_first = e.counters()
        e.reset()
        assert e.block_stats()[0] > 0
        again = e.run_to_stabilisation()
        assert again.values == first.values and again.modified == first.modified
        assert np.array_equal(e.counters(), c_first)
        e.reseed(8)
        other = e.run_to_stabilisation()
        c_other = e.counters()
    monkeypatch.setenv("HANF_BLOCK", "0")
    fresh = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=8))
    assert other.values == fresh.values and other.modified == fresh.modified
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=8)) as e:
        assert e.block_stats() == (0, 0)
        e.run_to_stabilisation()
        assert np.array_equal(e.counters(), c_other)


def test_blocked_restore_and_worklist(hanf, port, monkeypatch, tmp_path):
    """Restored counters restart the item rows; an engine whose CSR the
    worklist step already relabelled builds its items from row ids."""
    _force(monkeypatch, SHAPES[0])
    g = hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 6, 2)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=11)
    with hanf.NfEngine(g, cfg) as e:
        for _ in range(2):
            e.step()
        snap = tmp_path / "at2.hca"
        e.save_counters(snap)
        rest = []
        while True:
            rep = e.step()
            rest.append((rep.sum, rep.modified, e.counters()))
            if rep.modified == 0:
                break
        # a longer run's item rows must not leak into the restored state
        e.restore_counters(snap, iteration=2)
        for s_, m_, c_ in rest:
            rep = e.step()
            assert (rep.sum, rep.modified) == (s_, m_)
            assert np.array_equal(e.counters(), c_)
    _force(monkeypatch, SHAPES[0], mode="2")
    monkeypatch.setenv("HANF_SPARSE", "1")  # worklist steps: the CSR goes to row space
    g = hanf.gen_clique_path(600, 40)
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=3)) as e:
        first = e.run_to_stabilisation()
        e.reset()
        assert e.block_stats()[0] > 0
        again = e.run_to_stabilisation()
        assert again.values == first.values and again.modified == first.modified
    lockstep(hanf, port, g, bucket_bits=6, seed=3)


@pytest.mark.parametrize("chunk", ["1", "1000", "65536"])
def test_upload_maps_arc_chunks(hanf, port, monkeypatch, chunk):
    """Large relabelled engines upload the arcs in chunks and map each
    chunk's ids to rows under the rest of the upload (hanf_engine.cu
    create_engine; on by size from 2^26 arcs, forced here with tiny chunks):
    the plain sweeps, the worklist step (whose CSR rewrite then must not map
    again), the source-blocked sweeps and relabelled peer-push shards all
    read row ids and stay bit-exact; bad arc endpoints are still refused."""
    monkeypatch.setenv("HANF_RELABEL", "1")
    monkeypatch.setenv("HANF_MAP_CHUNK", chunk)
    for g in _graphs(hanf):
        lockstep(hanf, port, g, bucket_bits=6, seed=21)
    monkeypatch.setenv("HANF_SPARSE", "1")
    lockstep(hanf, port, hanf.gen_clique_path(600, 40), bucket_bits=6, seed=3)
    lockstep(hanf, port, hanf.gen_rmat(12, 16, 0.57, 0.19, 0.19, 6, 2), bucket_bits=7, seed=4)
    monkeypatch.delenv("HANF_SPARSE")
    _force(monkeypatch, SHAPES[0])
    for g in _graphs(hanf):
        lockstep(hanf, port, g, bucket_bits=6, seed=22)
    _force(monkeypatch, SHAPES[1], mode="2")
    monkeypatch.setenv("HANF_SPARSE", "1")
    g = hanf.gen_clique_path(600, 40)
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=3)) as e:
        first = e.run_to_stabilisation()
        e.reset()
        assert e.block_stats()[0] > 0
        again = e.run_to_stabilisation()
        assert again.values == first.values and again.modified == first.modified
    monkeypatch.delenv("HANF_SPARSE")
    monkeypatch.setenv("HANF_BLOCK", "0")
    bad = hanf.Graph(3, np.array([0, 1, 2, 2], dtype=np.uint64), np.array([1, 7], dtype=np.uint32))
    with pytest.raises(ValueError):
        hanf.NfEngine(bad, hanf.EngineConfig(bucket_bits=6, seed=1))
    import test_gpu_peer
    test_gpu_peer.test_peer_push_relabelled_shards(hanf, monkeypatch, 6, 4, True, False)
    monkeypatch.setenv("HANF_MAP_CHUNK", chunk)
    test_gpu_peer.test_peer_push_relabelled_shards(hanf, monkeypatch, 5, 2, True, True)
