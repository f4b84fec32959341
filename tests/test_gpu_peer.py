"""Peer-push exchange of sharded steps (hanf_shard_export / hanf_shard_attach,
include/hanf.h) on the one GPU a round has.

* In one process: 2 and 3 shard engines on cuda:0 attached with
  hanf_shard_attach_local.  Every union / worklist kernel stores its written
  rows into the other engines' next generation and publishes bitmap words
  and block sums; no exchange code runs on the host.  Computes run one after
  another and each finishes before the next begins (no kernel waits on
  another).  The schedule also lets a shard start step t+1 before another
  has committed step t - the case the per-generation block-sum inbox is
  for.  Equal to one engine bit for bit (N(t), modified, every counter).
* Across processes: 2 ranks on the same GPU, arenas mapped with CUDA IPC
  handles (hanf_shard_attach), ShardedNfEngine(exchange="peer") with a gloo
  barrier between compute and commit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run_local(hanf, g, cfg, world, skew, relabelled=False, reduce=False):
    import torch
    from paper_1011_5599_b200.sharded import LocalCudaShard, shard_ranges
    dev = torch.device("cuda", 0)
    shards = [LocalCudaShard(g, cfg, lo, hi, dev) for lo, hi in shard_ranges(g.num_nodes(), world)]
    engines = [sh.engine for sh in shards]
    assert all(bool(e.device_buffers().relabelled) == relabelled for e in engines)
    for k, e in enumerate(engines):
        e.shard_attach_local(engines, k)
    values, mods = [shards[0].sum_estimates()], [g.num_nodes()]
    pending = None  # skew: shard 0's commit of step t after shard 1's compute of t+1
    def computes(group):
        for sh in group:
            sh.shard_compute()
            sh.wait_compute()
        if reduce:  # (all computes of the step are done: the sliced block sums)
            for sh in shards:
                sh.shard_reduce()
                sh.wait_compute()

    while True:
        computes(shards)
        reps = [sh.shard_commit() for sh in shards[:1]] if skew else []
        if skew:
            # shard 0 runs ahead into its next compute (writes the other
            # generation of every peer's arena and block-sum inbox) before the
            # others commit this step
            if reps[0].modified:
                shards[0].shard_compute()
                shards[0].wait_compute()
                pending = True
            reps += [sh.shard_commit() for sh in shards[1:]]
        else:
            reps = [sh.shard_commit() for sh in shards]
        assert all(r.sum == reps[0].sum and r.modified == reps[0].modified for r in reps)
        if reps[0].modified == 0:
            break
        values.append(reps[0].sum)
        mods.append(reps[0].modified)
        if skew and pending:
            # the others now compute step t+1; shard 0 already did
            computes(shards[1:])
            reps = [sh.shard_commit() for sh in shards]
            assert all(r.sum == reps[0].sum and r.modified == reps[0].modified for r in reps)
            pending = None
            if reps[0].modified == 0:
                break
            values.append(reps[0].sum)
            mods.append(reps[0].modified)
    counters = [e.counters() for e in engines]
    for sh in shards:
        sh.shard_detach()
    for sh in shards:
        sh.close()
    return values, mods, counters


@pytest.mark.parametrize("b,env,world,skew", [
    (6, {}, 2, False), (6, {}, 3, False), (6, {}, 2, True), (6, {"HANF_SPARSE": "1"}, 2, False),
    (6, {"HANF_SPARSE": "1"}, 3, True), (5, {}, 2, True), (8, {}, 2, False), (7, {}, 3, False),
    (6, {"HANF_SEGMENTS": "1"}, 3, True), (5, {"HANF_SEGMENTS": "1", "HANF_SUMMARY": "1"}, 2, False)])
def test_peer_push_local(hanf, monkeypatch, b, env, world, skew):
    """Attached shard engines of one process: bit-exact with one engine, with
    the worklist step, the padded W = 3 rows, m = 128 and a multi-chunk layout."""
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    g = hanf.gen_rmat(14, 16, 0.57, 0.19, 0.19, 1, 7)
    cfg = hanf.EngineConfig(bucket_bits=b, seed=42)
    values, mods, counters = _run_local(hanf, g, cfg, world, skew)
    with hanf.NfEngine(g, cfg) as e:
        single = e.run_to_stabilisation()
        ref = e.counters()
    assert values == single.values and mods == single.modified
    for c in counters:
        assert np.array_equal(c, ref)


@pytest.mark.parametrize("b,world,skew,reduce", [
    (6, 2, False, False), (6, 4, True, False), (5, 2, True, False), (7, 4, False, False),
    (6, 4, False, True), (6, 4, True, True), (5, 2, True, True), (7, 4, False, True)])
def test_peer_push_relabelled_shards(hanf, monkeypatch, b, world, skew, reduce):
    """Relabelled shards (hanf_config.shard_count, degree order interleaved
    across the shards): rows live in another numbering on the device,
    estimates are pushed to the peers and every commit re-sums all
    original-id blocks.  N(t) and the counters equal one engine bit for bit."""
    import dataclasses
    monkeypatch.setenv("HANF_RELABEL", "1")
    g = hanf.gen_rmat(14, 16, 0.57, 0.19, 0.19, 1, 7)
    cfg = hanf.EngineConfig(bucket_bits=b, seed=42)
    values, mods, counters = _run_local(hanf, g, dataclasses.replace(cfg, shard_count=world),
                                        world, skew, relabelled=True, reduce=reduce)
    monkeypatch.setenv("HANF_RELABEL", "0")
    with hanf.NfEngine(g, cfg) as e:
        single = e.run_to_stabilisation()
        ref = e.counters()
    assert values == single.values and mods == single.modified
    for c in counters:
        assert np.array_equal(c, ref)


@pytest.mark.parametrize("need", ["1", "0"])
def test_peer_push_needed_rows_filter(hanf, monkeypatch, need):
    """Needed-rows filter of the peer push (hanf_shard_push_stats): after
    every step, each shard's pushed row stores equal the host count of its
    changed rows that each peer gathers (successors of the peer's nodes),
    and changed * peers with HANF_PEER_NEED=0.  The shards' changed rows
    are exactly the rows the single engine changed, and read-back (which
    pulls the peers' ranges) stays bit-exact."""
    import torch
    from paper_1011_5599_b200.sharded import LocalCudaShard, shard_ranges
    monkeypatch.setenv("HANF_PEER_NEED", need)
    g = hanf.gen_rmat(13, 8, 0.57, 0.19, 0.19, 1, 7)
    n, off, arcs = g.num_nodes(), g.offsets().astype(np.int64), g.arcs()
    cfg = hanf.EngineConfig(bucket_bits=6, seed=42)
    world = 3
    ranges = shard_ranges(n, world)
    needs = []
    for lo, hi in ranges:
        m = np.zeros(n, bool)
        m[arcs[off[lo]:off[hi]]] = True
        needs.append(m)
    dev = torch.device("cuda", 0)
    shards = [LocalCudaShard(g, cfg, lo, hi, dev) for lo, hi in ranges]
    engines = [sh.engine for sh in shards]
    for k, e in enumerate(engines):
        e.shard_attach_local(engines, k)
    total_pushed = total_all = 0
    with hanf.NfEngine(g, cfg) as single:
        prev = single.counters().reshape(n, -1)
        while True:
            for sh in shards:
                sh.shard_compute()
                sh.wait_compute()
            reps = [sh.shard_commit() for sh in shards]
            rep = single.step()
            assert all(r.sum == rep.sum and r.modified == rep.modified for r in reps)
            cur = single.counters().reshape(n, -1)
            changed = np.any(cur != prev, axis=1)
            prev = cur
            for k, ((lo, hi), e) in enumerate(zip(ranges, engines)):
                c, pushed = e.shard_push_stats()
                mine = changed[lo:hi]
                assert c == int(mine.sum())
                want = sum(int((mine & needs[p][lo:hi]).sum()) for p in range(world) if p != k)
                assert pushed == (want if need == "1" else c * (world - 1))
                total_pushed += want
                total_all += c * (world - 1)
            for e in engines:
                assert np.array_equal(e.counters().reshape(n, -1), cur)
            if rep.modified == 0:
                break
    assert total_pushed < total_all  # the filter has something to drop on R-MAT
    for sh in shards:
        sh.shard_detach()
    for sh in shards:
        sh.close()


def test_relabelled_shard_needs_peer_push(hanf, monkeypatch):
    import dataclasses
    import torch
    from paper_1011_5599_b200.sharded import LocalCudaShard, shard_ranges
    monkeypatch.setenv("HANF_RELABEL", "1")
    g = hanf.gen_rmat(12, 8, 0.57, 0.19, 0.19, 1, 7)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=1, shard_count=2)
    lo, hi = shard_ranges(g.num_nodes(), 2)[0]
    sh = LocalCudaShard(g, cfg, lo, hi, torch.device("cuda", 0))
    try:
        assert sh.engine.device_buffers().relabelled
        with pytest.raises(ValueError):
            sh.shard_compute()
    finally:
        sh.close()
    # unequal or unknown shards never relabel
    sh = LocalCudaShard(g, dataclasses.replace(cfg, shard_count=0), lo, hi, torch.device("cuda", 0))
    assert not sh.engine.device_buffers().relabelled
    sh.close()


def test_peer_attach_rejects_bad_peer_sets(hanf):
    import torch
    from paper_1011_5599_b200.sharded import LocalCudaShard, shard_ranges
    dev = torch.device("cuda", 0)
    g = hanf.gen_rmat(12, 8, 0.57, 0.19, 0.19, 1, 7)
    n = g.num_nodes()
    cfg = hanf.EngineConfig(bucket_bits=6, seed=1)
    a, b = [LocalCudaShard(g, cfg, lo, hi, dev) for lo, hi in shard_ranges(n, 2)]
    other = LocalCudaShard(g, hanf.EngineConfig(bucket_bits=7, seed=1), 0, n // 2, dev)
    try:
        with pytest.raises(ValueError):        # ranges do not tile [0, n)
            a.engine.shard_attach_local([a.engine, a.engine], 0)
        with pytest.raises(ValueError):        # self is not this engine
            a.engine.shard_attach_local([a.engine, b.engine], 1)
        with pytest.raises(ValueError):        # different counter layout
            other.engine.shard_attach_local([other.engine, b.engine], 0)
        exports = [a.engine.shard_export(), b.engine.shard_export()]
        with pytest.raises(ValueError):        # exports[self] must describe the engine
            a.engine.shard_attach(exports, 1)
    finally:
        for sh in (a, b, other):
            sh.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, out, relabel=False):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1011_5599_b200 as hanf
    from paper_1011_5599_b200.sharded import ShardedNfEngine
    torch.cuda.set_device(0)
    if relabel:
        os.environ["HANF_RELABEL"] = "1"
    g = hanf.gen_rmat(14, 16, 0.57, 0.19, 0.19, 1, 7)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=42)
    eng = ShardedNfEngine(g, cfg, rank, world, exchange="peer")
    assert eng.exchange == "peer", eng.fallback
    assert bool(eng.local.engine.device_buffers().relabelled) == relabel
    est = eng.run_to_stabilisation()
    out[rank] = (est.values, est.modified, eng.local.engine.counters())
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("relabel", [False, True])
def test_peer_push_ipc_two_processes(hanf, relabel):
    """Two ranks in two processes on one GPU, arenas mapped through CUDA IPC
    handles, ShardedNfEngine(exchange="peer"), plain and relabelled shards:
    equal to one engine."""
    import torch.multiprocessing as mp
    g = hanf.gen_rmat(14, 16, 0.57, 0.19, 0.19, 1, 7)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=42)
    with hanf.NfEngine(g, cfg) as e:
        single = e.run_to_stabilisation()
        ref = e.counters()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_ipc_worker, args=(2, _free_port(), out, relabel), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        values, mods, counters = out[r]
        assert values == single.values and mods == single.modified
        assert np.array_equal(counters, ref)


@pytest.mark.parametrize("relabel,world", [("0", 2), ("1", 4)])
def test_peer_push_config2_full_size(hanf, monkeypatch, relabel, world):
    """BASELINE config 2 at full size (R-MAT 20, 16.1 M arcs) as 2 / 4
    peer-push shards on one GPU, plain and relabelled: N(t), modified and
    every counter equal to the single engine's."""
    import dataclasses
    monkeypatch.setenv("HANF_RELABEL", relabel)
    g = hanf.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=42)
    values, mods, counters = _run_local(hanf, g, dataclasses.replace(cfg, shard_count=world),
                                        world, False, relabelled=relabel == "1",
                                        reduce=relabel == "1")
    monkeypatch.setenv("HANF_RELABEL", "0")
    with hanf.NfEngine(g, cfg) as e:
        single = e.run_to_stabilisation()
        ref = e.counters()
    assert values == single.values and mods == single.modified
    for c in counters:
        assert np.array_equal(c, ref)


@pytest.mark.parametrize("world,hot", [(2, "0"), (4, "64")])
def test_peer_push_relabelled_shards_line_slots(hanf, monkeypatch, world, hot):
    """Relabelled shards with the reference packing (W = 5 rows) and the
    line-aligned slot assignment inside every shard range forced small
    (by default only past 2^22 / G rows): bit for bit against one engine."""
    import dataclasses
    monkeypatch.setenv("HANF_LAYOUT", "packed")
    monkeypatch.setenv("HANF_RELABEL", "1")
    monkeypatch.setenv("HANF_SLOTS_HOT", hot)
    g = hanf.gen_rmat(14, 16, 0.57, 0.19, 0.19, 1, 7)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=42)
    values, mods, counters = _run_local(hanf, g, dataclasses.replace(cfg, shard_count=world),
                                        world, True, relabelled=True, reduce=True)
    monkeypatch.setenv("HANF_RELABEL", "0")
    with hanf.NfEngine(g, cfg) as e:
        single = e.run_to_stabilisation()
        ref = e.counters()
    assert values == single.values and mods == single.modified
    for c in counters:
        assert np.array_equal(c, ref)
