"""Node-range sharding of the HyperANF iteration across GPUs (one process per
GPU, torch.distributed for the plumbing).

Every rank holds the full previous generation (successor gathers are
random), computes the next generation for its contiguous node range, and
the shards are exchanged once per iteration: the next-generation counter
rows, the "modified" bitmap words and the 64-counter block sums.  Each
rank then reduces N(t) and the modified count over the full arrays, so all
ranks agree on the report without a separate all-reduce.  Exchange = an
in-place all-gather when the shards are equal (n a multiple of 64*world),
else one broadcast per owner.

Late iterations change few counters, so once the previous step changed
fewer than n/16 of them the counter shards travel as changed rows only
(hanf_shard_pack / hanf_shard_unpack): each owner packs the rows its step
wrote - the only rows in which the peers' copies differ - and every rank
scatters the other ranks' packets.  Bitmaps and block sums still travel
whole (they are 1/(8*40) of the counters).

Peer-push exchange (exchange="peer", hanf_shard_attach): the shard
engines map each other's exchange arenas (CUDA IPC handles, all-gathered
once) and the union / worklist kernels store every row they write straight
into the peers' next generation over NVLink while the sweep runs; a last
kernel publishes the shard's bitmap words and block sums.  A step is then
compute -> wait for the engine stream -> barrier -> commit: no counter
bytes go through a collective and unchanged rows are never sent.  Block
sums land in a per-generation inbox, so one barrier per step suffices (a
fast rank's step t+1 never overwrites what a slow rank's commit t reads).

The local engine is anything with shard_compute() / exchange_buffers() /
shard_commit() / before_exchange() / after_exchange() and optionally
pack_rows() / unpack_rows(): the CUDA engine (`LocalCudaShard`) in
production, a CPU emulation in the gloo tests.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

import torch
import torch.distributed as dist

from .engine import EngineConfig, IterationReport, NfEngine, NfEstimate


def shard_ranges(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous node ranges, each a multiple of 64 nodes (the last one may
    be short or empty), so bitmap words and block sums split cleanly."""
    per = -(-n // world) if world else n
    per = -(-per // 64) * 64
    return [(min(k * per, n), min((k + 1) * per, n)) for k in range(world)]


class _CudaArray:
    """Minimal __cuda_array_interface__ holder for a raw device pointer."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3,
                                         "strides": None}


def device_tensor(ptr: int, count: int, dtype: torch.dtype, device: torch.device):
    typestr = {torch.int64: "<i8", torch.float64: "<f8"}[dtype]
    return torch.as_tensor(_CudaArray(ptr, count, typestr), device=device)


class LocalCudaShard:
    """The CUDA engine restricted to one node range."""

    def __init__(self, graph, cfg: EngineConfig, lo: int, hi: int, device: torch.device):
        self.engine = NfEngine(graph, dataclasses.replace(cfg, shard_begin=lo, shard_end=hi))
        self.n = graph.num_nodes()
        self.device = device
        self.stream = torch.cuda.ExternalStream(self.engine.stream(), device=device)

    def shard_compute(self):
        self.engine.shard_compute()

    def before_exchange(self):
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def after_exchange(self):
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def exchange_buffers(self):
        """(full tensor, elements per 64-node unit) for the three buffers the
        next commit reads; the generation flips every step, so re-fetch."""
        b = self.engine.device_buffers()
        blocks = int(b.blocks)
        W = int(b.row_pitch)  # u64 words per counter row on the device (>= W)
        counters = device_tensor(b.next_counters, self.n * W, torch.int64, self.device)
        modified = device_tensor(b.next_modified, blocks, torch.int64, self.device)
        sums = device_tensor(b.block_sums, blocks, torch.float64, self.device)
        return [(counters, 64 * W, W), (modified, 1, None), (sums, 1, None)]

    def shard_commit(self) -> IterationReport:
        return self.engine.shard_commit()

    # peer-push exchange
    def shard_export(self) -> bytes:
        return self.engine.shard_export()

    def shard_attach(self, exports, rank: int) -> None:
        self.engine.shard_attach(exports, rank)

    def shard_detach(self) -> None:
        self.engine.shard_detach()

    def needs_reduce(self) -> bool:
        return bool(self.engine.device_buffers().relabelled)

    def shard_reduce(self) -> None:
        self.engine.shard_reduce()

    def wait_compute(self) -> None:
        self.stream.synchronize()

    def row_words(self) -> int:
        return int(self.engine.device_buffers().row_pitch)

    def pack_rows(self, ids: torch.Tensor, rows: torch.Tensor) -> int:
        """Changed rows of this shard into ids (int32) / rows (int64); -1 when
        more than ids.numel() rows changed."""
        import ctypes
        from ctypes import c_uint64, c_void_p
        from ._lib import CAPACITY, check, lib
        cnt = c_uint64()
        st = lib().hanf_shard_pack(self.engine._h, c_void_p(ids.data_ptr()),
                                   c_void_p(rows.data_ptr()), ids.numel(), ctypes.byref(cnt))
        if st == CAPACITY:
            return -1
        check(st)
        return int(cnt.value)

    def unpack_rows(self, ids: torch.Tensor, rows: torch.Tensor, count: int) -> None:
        from ctypes import c_void_p
        from ._lib import check, lib
        self.stream.wait_stream(torch.cuda.current_stream(self.device))  # the gathered packets
        check(lib().hanf_shard_unpack(self.engine._h, c_void_p(ids.data_ptr()),
                                      c_void_p(rows.data_ptr()), count))

    def new_buffer(self, count: int, dtype: torch.dtype) -> torch.Tensor:
        return torch.empty(count, dtype=dtype, device=self.device)

    def sum_estimates(self) -> float:
        return self.engine.sum_estimates()

    def close(self):
        self.engine.close()


class ShardedNfEngine:
    """NfEngine across `world` ranks (engine.hpp:122-275 semantics)."""

    def __init__(self, graph, cfg: EngineConfig, rank: int, world: int, local=None,
                 group=None, delta: bool = True, delta_ratio: int = 16, delta_cap: int = None,
                 exchange: str = "collective"):
        self.n = graph.num_nodes()
        self.cfg = cfg
        self.rank, self.world, self.group = rank, world, group
        self.ranges = shard_ranges(self.n, world)
        lo, hi = self.ranges[rank]
        own_local = local is None
        if own_local:
            # peer-push shards may relabel (hanf_config.shard_count)
            local = LocalCudaShard(graph, dataclasses.replace(
                cfg, shard_count=world if exchange == "peer" else 0), lo, hi,
                torch.device("cuda", torch.cuda.current_device()))
        self.local = local
        if exchange not in ("collective", "peer"):
            raise ValueError(f"exchange must be 'collective' or 'peer', not {exchange!r}")
        self.exchange = exchange
        self.fallback = None
        self.sliced = False
        if exchange == "peer":
            # every rank's arena description, then map the others' arenas;
            # if any rank cannot map a peer (no IPC / peer access between
            # the devices) all ranks fall back to the collective exchange
            exports = [None] * world
            dist.all_gather_object(exports, local.shard_export(), group=group)
            error = None
            try:
                local.shard_attach(exports, rank)
            except Exception as exc:  # noqa: BLE001 - reported through self.fallback
                error = f"rank {rank}: {exc}"
            errors = [None] * world
            dist.all_gather_object(errors, error, group=group)
            errors = [e for e in errors if e]
            self.fallback = errors[0] if errors else None
            if errors:
                if error is None:
                    local.shard_detach()
                dist.barrier(group=group)  # no rank maps an arena that is freed next
                self.exchange = "collective"
                if own_local:  # (a relabelled shard needs the peer-push exchange)
                    local.close()
                    self.local = local = LocalCudaShard(
                        graph, cfg, lo, hi, torch.device("cuda", torch.cuda.current_device()))
        self.sliced = (self.exchange == "peer" and hasattr(local, "needs_reduce")
                       and local.needs_reduce())
        # changed-rows exchange (see the module docstring); packets hold at
        # most n/16 rows
        self.delta = delta and hasattr(local, "pack_rows")
        self.delta_ratio = delta_ratio  # changed rows once ratio * modified < n
        self.last_modified = self.n
        self.delta_steps = 0
        if self.delta:
            self.cap = delta_cap or max(64, self.n // 16)
            self.words = local.row_words()
            self.ids = local.new_buffer(self.cap, torch.int32)
            self.rows = local.new_buffer(self.cap * self.words, torch.int64)

    def _exchange(self, tensor: torch.Tensor, unit: int, per_node):
        """Gives every rank the owners' slices of `tensor`.  unit = elements
        per 64 nodes; per_node = elements per node (counters) or None."""
        spans = []
        for lo, hi in self.ranges:
            if per_node is not None:
                spans.append((lo * per_node, hi * per_node))
            else:
                spans.append((lo // 64, -(-hi // 64)))
        sizes = [e - b for b, e in spans]
        if len(set(sizes)) == 1 and spans[-1][1] == tensor.numel():
            dist.all_gather_into_tensor(tensor, tensor[spans[self.rank][0]:spans[self.rank][1]],
                                        group=self.group)
        else:
            for k, (b, e) in enumerate(spans):
                if e > b:
                    view = tensor[b:e]
                    dist.broadcast(view, src=k, group=self.group)

    def _exchange_changed_rows(self) -> bool:
        """Changed-rows exchange of the counters; False when some shard had
        more than `cap` rows (the caller then exchanges whole shards)."""
        count = self.local.pack_rows(self.ids, self.rows)
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
        mine = torch.tensor([count], dtype=torch.int64)
        if self.ids.is_cuda:
            counts = [c.to(self.ids.device) for c in counts]
            mine = mine.to(self.ids.device)
        dist.all_gather(counts, mine, group=self.group)
        counts = [int(c.item()) for c in counts]
        if min(counts) < 0:
            return False
        m = max(counts)
        if m == 0:
            return True
        self.ids[count:m] = -1  # padding: ids >= n are skipped by the unpack
        ids_all = [torch.empty_like(self.ids[:m]) for _ in range(self.world)]
        rows_all = [torch.empty_like(self.rows[:m * self.words]) for _ in range(self.world)]
        dist.all_gather(ids_all, self.ids[:m].contiguous(), group=self.group)
        dist.all_gather(rows_all, self.rows[:m * self.words].contiguous(), group=self.group)
        for k in range(self.world):
            if k != self.rank and counts[k]:
                self.local.unpack_rows(ids_all[k], rows_all[k], counts[k])
        return True

    def step(self) -> IterationReport:
        if self.n == 0:
            return IterationReport(0.0, 0)
        self.local.shard_compute()
        if self.exchange == "peer":
            # the kernels pushed rows, bitmap words and block sums into the
            # peers' arenas: once every rank's compute is done, commit
            self.local.wait_compute()
            dist.barrier(group=self.group)
            if self.sliced:
                # relabelled shards: each rank re-sums 1/world of the blocks
                # and publishes them, instead of every rank re-summing all
                self.local.shard_reduce()
                self.local.wait_compute()
                dist.barrier(group=self.group)
            rep = self.local.shard_commit()
            self.last_modified = rep.modified
            return rep
        self.local.before_exchange()
        rows_done = False
        if self.delta and self.delta_ratio * self.last_modified < self.n:
            rows_done = self._exchange_changed_rows()
            self.delta_steps += rows_done
        for tensor, unit, per_node in self.local.exchange_buffers():
            if per_node is not None and rows_done:
                continue  # the counters went as changed rows
            self._exchange(tensor, unit, per_node)
        self.local.after_exchange()
        rep = self.local.shard_commit()
        self.last_modified = rep.modified
        return rep

    def sum_estimates(self) -> float:
        return self.local.sum_estimates()

    def reset(self) -> None:
        """hanf_reset on every rank, then a barrier: with the peer-push
        exchange a rank that started its next step could otherwise push rows
        into a peer that is still re-seeding both generations."""
        self.local.engine.reset()
        self.local.wait_compute()
        dist.barrier(group=self.group)
        self.last_modified = self.n

    def run_to_stabilisation(self) -> NfEstimate:
        """engine.hpp:233-275 over the sharded step."""
        est = NfEstimate(n=self.n, m=1 << self.cfg.bucket_bits, seed=self.cfg.seed,
                         termination=self.cfg.termination)
        if self.n == 0:
            return est
        cap = self.cfg.max_iterations or (self.n + 1)
        est.values.append(self.sum_estimates())
        est.modified.append(self.n)
        while True:
            if len(est.values) - 1 >= cap:
                from ._lib import GuardError
                raise GuardError(f"engine: iteration cap {cap} exceeded; pathological input or bug")
            rep = self.step()
            if rep.modified == 0:
                break
            prev = est.values[-1]
            est.values.append(rep.sum)
            est.modified.append(rep.modified)
            if int(self.cfg.termination) == 1 and prev > 0.0:
                if (rep.sum - prev) / prev < self.cfg.eps_inc:
                    break
        for t in range(1, len(est.values)):
            est.values[t] = max(est.values[t], est.values[t - 1])
        return est

    def close(self):
        if self.exchange == "peer":
            # unmap the peers' arenas before any owner frees its own
            self.local.shard_detach()
            dist.barrier(group=self.group)
        self.local.close()
