"""Multi-rank path on CPU: ShardedNfEngine (paper_1011_5599_b200/sharded.py)
over torch.distributed/gloo with world_size 2 and 3, each rank driving a CPU
emulation of one CUDA shard engine (same buffers, same exchange contract).
The sharded run must equal the single-engine reference run bit for bit."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


class EmulatedShard:
    """CPU stand-in for LocalCudaShard: next-generation rows of [lo, hi),
    the modified bitmap words and 64-counter block sums, exchanged by the
    orchestrator, then a commit over the full arrays (hanf_engine.cu
    compute_local/commit semantics, arithmetic from the oracle)."""

    def __init__(self, graph, cfg, lo, hi):
        import oracle
        self.port = oracle.port()
        self.n = graph.num_nodes()
        self.off, self.succ = graph.offsets(), graph.arcs()
        self.lo, self.hi = lo, hi
        r = cfg.register_bits or 5
        self.p = self.port.params(cfg.bucket_bits, cfg.seed, r)
        W = self.p.words
        self.W = W
        self.cur = np.zeros((self.n, W), dtype=np.uint64)
        for v in range(self.n):
            self.cur[v] = self.port.counter_of(self.p, [v])
        self.next = self.cur.copy()
        nb = (self.n + 63) // 64
        self.mod_cur = np.zeros(nb, dtype=np.uint64)
        self.mod_next = np.zeros(nb, dtype=np.uint64)
        self.est = np.array([self.port.estimate(self.cur[v], self.p) for v in range(self.n)])
        self.block_sums = np.zeros(nb)
        for b in range(nb):
            s = 0.0
            for v in range(64 * b, min(64 * b + 64, self.n)):
                s += self.est[v]
            self.block_sums[b] = s
        self.t = 0
        self.last_sum = float(np.sum(self.block_sums[:0]))
        self.last_sum = self._total()

    def _total(self):
        s = 0.0
        for x in self.block_sums:
            s += x
        return s

    def sum_estimates(self):
        return self.last_sum

    def shard_compute(self):
        lo, hi = self.lo, self.hi
        self.mod_next[lo // 64:-(-hi // 64)] = 0
        for v in range(lo, hi):
            acc = self.cur[v].copy()
            for i in range(int(self.off[v]), int(self.off[v + 1])):
                self.port.packed_max_into(self.p, acc, np.ascontiguousarray(self.cur[self.succ[i]]))
            self.next[v] = acc
            if not np.array_equal(acc, self.cur[v]):
                self.mod_next[v >> 6] |= np.uint64(1) << np.uint64(v & 63)
                self.est[v] = self.port.estimate(acc, self.p)
        for b in range(lo // 64, -(-hi // 64)):
            if self.mod_next[b]:
                s = 0.0
                for v in range(64 * b, min(64 * b + 64, self.n)):
                    s += self.est[v]
                self.block_sums[b] = s

    def before_exchange(self):
        pass

    def after_exchange(self):
        pass

    def exchange_buffers(self):
        counters = torch.from_numpy(self.next.reshape(-1).view(np.int64))
        modified = torch.from_numpy(self.mod_next.view(np.int64))
        sums = torch.from_numpy(self.block_sums)
        return [(counters, 64 * self.W, self.W), (modified, 1, None), (sums, 1, None)]

    # changed-rows exchange (LocalCudaShard.pack_rows / unpack_rows contract)
    def row_words(self):
        return self.W

    def new_buffer(self, count, dtype):
        return torch.zeros(count, dtype=dtype)

    def pack_rows(self, ids, rows):
        lo, hi = self.lo, self.hi
        picked = [v for v in range(lo, hi)
                  if (int(self.mod_next[v >> 6]) | int(self.mod_cur[v >> 6])) >> (v & 63) & 1]
        if len(picked) > ids.numel():
            return -1
        for i, v in enumerate(picked):
            ids[i] = v
            rows[i * self.W:(i + 1) * self.W] = torch.from_numpy(self.next[v].view(np.int64))
        return len(picked)

    def unpack_rows(self, ids, rows, count):
        for i in range(count):
            v = int(ids[i]) & 0xFFFFFFFF
            if v < self.n:
                self.next[v] = rows[i * self.W:(i + 1) * self.W].numpy().view(np.uint64)

    def shard_commit(self):
        from paper_1011_5599_b200.engine import IterationReport
        count = int(sum(bin(int(w)).count("1") for w in self.mod_next))
        total = self._total()
        self.cur, self.next = self.next, self.cur.copy()
        self.next[:] = self.cur
        self.mod_cur, self.mod_next = self.mod_next, self.mod_cur
        self.t += 1
        self.last_sum = total
        return IterationReport(total, count)

    def close(self):
        pass


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _drop_rendezvous(tag):
    try:
        os.unlink(f"/tmp/hanf_gloo_{os.getpid()}_{tag}")
    except FileNotFoundError:
        pass


def _fresh_tag():
    """A tag unique to this run (also names the emulated peers' shared
    memory), with no rendezvous file left over from an earlier run."""
    tag = _free_port()
    _drop_rendezvous(tag)
    return tag


def _worker(rank, world, port, spec, out):
    import sys
    sys.path.insert(0, ROOT)
    # file rendezvous: a TCP port picked by the parent can be taken again
    # before the workers bind it (`port` stays the run's unique tag)
    dist.init_process_group("gloo", init_method=f"file:///tmp/hanf_gloo_{os.getppid()}_{port}",
                            rank=rank, world_size=world)
    import paper_1011_5599_b200 as hanf
    from paper_1011_5599_b200.sharded import ShardedNfEngine, shard_ranges
    g = hanf.gen_uniform_random(*spec["graph"])
    cfg = hanf.EngineConfig(bucket_bits=spec["b"], seed=spec["seed"])
    lo, hi = shard_ranges(g.num_nodes(), world)[rank]
    eng = ShardedNfEngine(g, cfg, rank, world, local=EmulatedShard(g, cfg, lo, hi),
                          delta=spec.get("delta", True), delta_ratio=2, delta_cap=g.num_nodes())
    est = eng.run_to_stabilisation()
    out[rank] = (est.values, est.modified, eng.local.cur.copy(), eng.delta_steps)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,graph,delta", [(2, (256, 4, 5), True), (3, (200, 3, 9), True),
                                               (2, (130, 2, 1), True), (2, (256, 4, 5), False)])
def test_sharded_run_matches_single_engine(port, world, graph, delta):
    spec = {"graph": graph, "b": 6, "seed": 42, "delta": delta}
    mgr = mp.Manager()
    out = mgr.dict()
    tag = _fresh_tag()
    mp.start_processes(_worker, args=(world, tag, spec, out), nprocs=world,
                       join=True, start_method="spawn")
    _drop_rendezvous(tag)
    n, off, succ = port.gen_uniform_random(*graph)
    vals, mods = port.engine(n, off, succ, bucket_bits=6, seed=42).run()
    final = port.engine(n, off, succ, bucket_bits=6, seed=42)
    while final.step()[1]:
        pass
    for r in range(world):
        v, m, cur, delta_steps = out[r]
        assert v == vals and m == mods
        assert np.array_equal(cur.reshape(-1), final.counters())
        assert (delta_steps > 0) == delta  # the tail went as changed rows


def test_shard_ranges():
    from paper_1011_5599_b200.sharded import shard_ranges
    assert shard_ranges(1 << 20, 8) == [(k << 17, (k + 1) << 17) for k in range(8)]
    r = shard_ranges(1000, 3)
    assert r[0][0] == 0 and r[-1][1] == 1000
    assert all(lo % 64 == 0 for lo, _ in r)
    assert all(r[i][1] == r[i + 1][0] for i in range(2))
    assert shard_ranges(10, 4)[1:] == [(10, 10)] * 3


class EmulatedPeerShard:
    """CPU stand-in for a LocalCudaShard attached with hanf_shard_attach
    (peer-push exchange).  Each rank's exchange arena - both counter
    generations, both modified bitmaps, both block-sum inboxes - lives in
    shared memory; compute writes only the rows that changed or are stale
    (the engine's stale-slot invariant) and stores each of them into every
    peer's next generation too, then publishes its bitmap words and block
    sums (hanf_engine.cu compute_local / publish_kernel / finish_enqueue).
    `lag` sleeps before reading the inbox in commit, so a fast rank's step
    t+1 publishes while a slow rank still commits step t."""

    def __init__(self, graph, cfg, lo, hi, tag, lag=0.0):
        from multiprocessing import shared_memory
        import oracle
        self.port = oracle.port()
        self.n = graph.num_nodes()
        self.off, self.succ = graph.offsets(), graph.arcs()
        self.lo, self.hi, self.lag = lo, hi, lag
        r = cfg.register_bits or 5
        self.p = self.port.params(cfg.bucket_bits, cfg.seed, r)
        self.W = W = self.p.words
        self.nb = nb = (self.n + 63) // 64
        self.layout = [(2, (self.n, W), np.uint64), (2, (nb,), np.uint64), (2, (nb,), np.float64)]
        self.bytes = 2 * (self.n * W * 8) + 2 * nb * 8 + 2 * nb * 8
        self.name = f"hanf_{tag}_{lo}"
        self.shm = shared_memory.SharedMemory(name=self.name, create=True, size=max(8, self.bytes))
        self.cnt, self.mod, self.inbox = self._views(self.shm)
        seeded = np.stack([self.port.counter_of(self.p, [v]) for v in range(self.n)])
        self.cnt[0][:] = seeded
        self.cnt[1][:] = seeded
        self.mod[0][:] = 0
        for v in range(self.n):                      # launch_seed_bitmap: all modified
            self.mod[0][v >> 6] |= np.uint64(1) << np.uint64(v & 63)
        self.est = np.array([self.port.estimate(seeded[v], self.p) for v in range(self.n)])
        self.block_sums = np.array([self._block(b) for b in range(nb)])
        self.g, self.stale_valid, self.peers = 0, False, []
        self.last_sum = 0.0
        for x in self.block_sums:
            self.last_sum += x

    def _views(self, shm):
        n, W, nb = self.n, self.W, self.nb
        buf, at = shm.buf, 0
        cnt, mod, inbox = [], [], []
        for _ in range(2):
            cnt.append(np.ndarray((n, W), np.uint64, buf, at)); at += n * W * 8
        for _ in range(2):
            mod.append(np.ndarray((nb,), np.uint64, buf, at)); at += nb * 8
        for _ in range(2):
            inbox.append(np.ndarray((nb,), np.float64, buf, at)); at += nb * 8
        return cnt, mod, inbox

    def _block(self, b):
        s = 0.0
        for v in range(64 * b, min(64 * b + 64, self.n)):
            s += self.est[v]
        return s

    def sum_estimates(self):
        return self.last_sum

    def shard_export(self):
        return (self.name, self.lo, self.hi)

    def shard_attach(self, exports, rank):
        from multiprocessing import shared_memory
        from multiprocessing import resource_tracker
        for k, (name, lo, hi) in enumerate(exports):
            if k != rank:
                shm = shared_memory.SharedMemory(name=name)
                resource_tracker.unregister(shm._name, "shared_memory")  # owner unlinks
                self.peers.append((shm, self._views(shm)))

    def shard_compute(self):
        g, ng = self.g, 1 - self.g
        cur, nxt = self.cnt[g], self.cnt[ng]
        w0, w1 = self.lo // 64, -(-self.hi // 64)
        self.mod[ng][w0:w1] = 0
        for v in range(self.lo, self.hi):
            acc = cur[v].copy()
            for i in range(int(self.off[v]), int(self.off[v + 1])):
                self.port.packed_max_into(self.p, acc, np.ascontiguousarray(cur[self.succ[i]]))
            changed = not np.array_equal(acc, cur[v])
            stale = self.stale_valid and (int(self.mod[g][v >> 6]) >> (v & 63)) & 1
            if changed or stale:
                nxt[v] = acc
                for _, (pc, _, _) in self.peers:
                    pc[ng][v] = acc
            if changed:
                self.mod[ng][v >> 6] |= np.uint64(1) << np.uint64(v & 63)
                self.est[v] = self.port.estimate(acc, self.p)
        for b in range(w0, w1):
            if self.mod[ng][b]:
                self.block_sums[b] = self._block(b)
        for _, (_, pm, pi) in self.peers:            # publish_kernel
            pm[ng][w0:w1] = self.mod[ng][w0:w1]
            pi[ng][w0:w1] = self.block_sums[w0:w1]
        self.inbox[ng][w0:w1] = self.block_sums[w0:w1]

    def wait_compute(self):
        pass

    def shard_commit(self):
        import time
        from paper_1011_5599_b200.engine import IterationReport
        if self.lag:
            time.sleep(self.lag)
        ng = 1 - self.g
        count = int(sum(bin(int(w)).count("1") for w in self.mod[ng]))
        total = 0.0
        for x in self.inbox[ng]:
            total += x
        self.g, self.stale_valid = ng, True
        self.last_sum = total
        return IterationReport(total, count)

    def counters(self):
        return self.cnt[self.g].copy()

    def shard_detach(self):
        for shm, _ in self.peers:
            shm.close()
        self.peers = []

    def close(self):
        self.cnt = self.mod = self.inbox = None
        self.shm.close()
        self.shm.unlink()


def _peer_worker(rank, world, port, spec, out):
    import sys
    sys.path.insert(0, ROOT)
    # file rendezvous: a TCP port picked by the parent can be taken again
    # before the workers bind it (`port` stays the run's unique tag)
    dist.init_process_group("gloo", init_method=f"file:///tmp/hanf_gloo_{os.getppid()}_{port}",
                            rank=rank, world_size=world)
    import paper_1011_5599_b200 as hanf
    from paper_1011_5599_b200.sharded import ShardedNfEngine, shard_ranges
    g = hanf.gen_uniform_random(*spec["graph"])
    cfg = hanf.EngineConfig(bucket_bits=spec["b"], seed=spec["seed"])
    lo, hi = shard_ranges(g.num_nodes(), world)[rank]
    local = EmulatedPeerShard(g, cfg, lo, hi, tag=port, lag=0.05 if rank == 0 else 0.0)
    eng = ShardedNfEngine(g, cfg, rank, world, local=local, exchange="peer")
    est = eng.run_to_stabilisation()
    out[rank] = (est.values, est.modified, local.counters())
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,graph", [(2, (256, 4, 5)), (3, (200, 3, 9))])
def test_peer_push_run_matches_single_engine(port, world, graph):
    """Peer-push protocol (rows pushed by the compute, one barrier per step,
    double-buffered block sums) with a lagging rank: equal to one engine."""
    spec = {"graph": graph, "b": 6, "seed": 42}
    mgr = mp.Manager()
    out = mgr.dict()
    tag = _fresh_tag()
    mp.start_processes(_peer_worker, args=(world, tag, spec, out), nprocs=world,
                       join=True, start_method="spawn")
    _drop_rendezvous(tag)
    n, off, succ = port.gen_uniform_random(*graph)
    vals, mods = port.engine(n, off, succ, bucket_bits=6, seed=42).run()
    final = port.engine(n, off, succ, bucket_bits=6, seed=42)
    while final.step()[1]:
        pass
    for r in range(world):
        v, m, cur = out[r]
        assert v == vals and m == mods
        assert np.array_equal(cur.reshape(-1), final.counters())


def test_peer_exchange_mode_is_checked():
    from paper_1011_5599_b200.sharded import ShardedNfEngine
    import paper_1011_5599_b200 as hanf
    g = hanf.gen_uniform_random(64, 2, 1)
    with pytest.raises(ValueError):
        ShardedNfEngine(g, hanf.EngineConfig(), 0, 1, local=object(), exchange="nvshmem")
