"""Peer-push volume of G relabelled shards of R-MAT `scale` on one GPU
(hanf_shard_attach_local; computes in sequence), with and without the
needed-rows filter (HANF_PEER_NEED): per step, the rows each shard changed,
the row stores it pushed to peers (hanf_shard_push_stats), and the union
sweep per shard.  On one GPU the pushed rows land in local HBM, so the
sweep time also shows the store side of the push.

  python scripts/peer_push_volume.py [scale] [G] [steps]
"""
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1011_5599_b200 as hanf  # noqa: E402
from paper_1011_5599_b200.sharded import LocalCudaShard, shard_ranges  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
t0 = time.time()
g = hanf.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
n = g.num_nodes()
print(f"R-MAT {scale}: n={n} arcs={g.num_arcs()} ({time.time() - t0:.1f} s), G={G}", flush=True)
cfg = hanf.EngineConfig(bucket_bits=6, seed=42, exact_sum=False, shard_count=G)
dev = torch.device("cuda", 0)
os.environ["HANF_RELABEL"] = "1"

results = {}
for need in ("0", "1"):
    os.environ["HANF_PEER_NEED"] = need
    shards = [LocalCudaShard(g, cfg, lo, hi, dev) for lo, hi in shard_ranges(n, G)]
    engines = [s.engine for s in shards]
    for k, e in enumerate(engines):
        e.shard_attach_local(engines, k)
        e.set_timing(True)
    row = 8 * int(engines[0].device_buffers().row_pitch)
    per_step = []
    for t in range(1, steps + 1):
        before = [e.timing()["union_ms"] for e in engines]
        for s in shards:
            s.shard_compute()
            s.wait_compute()
        for s in shards:
            s.shard_reduce()
            s.wait_compute()
        reps = [s.shard_commit() for s in shards]
        stats = [e.shard_push_stats() for e in engines]
        union = [e.timing()["union_ms"] - b for e, b in zip(engines, before)]
        changed = sum(c for c, _ in stats)
        pushed = sum(p for _, p in stats)
        per_step.append((reps[0].sum, reps[0].modified, changed, pushed, max(union),
                         sum(union) / G))
        print(f"need={need} t={t}: modified {reps[0].modified}, changed rows {changed}, "
              f"row stores pushed {pushed} ({pushed / max(1, changed * (G - 1)):.3f} of "
              f"changed x (G-1)), max per shard {max(p for _, p in stats) * row / 1e9:.3f} GB; "
              f"union per shard max {max(union):.3f} mean {sum(union) / G:.3f} ms", flush=True)
        if reps[0].modified == 0:
            break
    results[need] = per_step
    for s in shards:
        s.shard_detach()
    for s in shards:
        s.close()

same = all(a[:2] == b[:2] for a, b in zip(results["0"], results["1"]))
print(f"N(t), modified identical with and without the filter: {same}", flush=True)
