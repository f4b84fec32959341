"""Per-shard union sweep of G peer-push shards of one graph on one GPU
(hanf_shard_attach_local; computes in sequence), relabelled vs plain, next
to the single engine.  On one GPU the peers' rows land in local HBM, so
every shard also writes G-1 extra copies of its changed rows: an upper
bound on the store side of the NVLink push.

  python scripts/shard_relabel_time.py [scale] [G]
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
t0 = time.time()
g = hanf.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
print(f"R-MAT {scale}: n={g.num_nodes()} arcs={g.num_arcs()} ({time.time() - t0:.1f} s)", flush=True)
cfg = hanf.EngineConfig(bucket_bits=6, seed=42, exact_sum=False)
dev = torch.device("cuda", 0)


def single(relabel):
    os.environ["HANF_RELABEL"] = "1" if relabel else "0"
    with hanf.NfEngine(g, cfg) as e:
        e.set_timing(True)
        e.step()
        e.step()
        t = e.timing()
    return t["union_ms"] / t["steps"], t["reduce_ms"] / t["steps"]


def sharded(relabel, scatter="1"):
    os.environ["HANF_RELABEL"] = "1" if relabel else "0"
    c = dataclasses.replace(cfg, shard_count=G)
    shards = [LocalCudaShard(g, c, lo, hi, dev) for lo, hi in shard_ranges(g.num_nodes(), G)]
    engines = [s.engine for s in shards]
    for k, e in enumerate(engines):
        e.shard_attach_local(engines, k)
        e.set_timing(True)
    rows = []
    steps = int(os.environ.get("STEPS", "2"))  # 0: to stabilisation
    red = [0.0] * G
    sliced = relabel and os.environ.get("SLICED", "1") == "1"
    while True:
        for s in shards:
            s.shard_compute()
            s.wait_compute()
        if sliced:  # hanf_shard_reduce: each shard re-sums 1/G of the blocks
            for k, s in enumerate(shards):
                t0 = time.perf_counter()
                s.shard_reduce()
                s.wait_compute()
                red[k] += 1e3 * (time.perf_counter() - t0)
        reps = [s.shard_commit() for s in shards]
        rows.append(reps[0])
        if reps[0].modified == 0 or (steps and len(rows) >= steps):
            break
    if not steps:
        t = [e.timing() for e in engines]
        print(f"   whole run: {len(rows)} steps, union per shard {max(x['union_ms'] for x in t):.2f} ms, "
              f"finish per shard {max(x['reduce_ms'] for x in t):.2f} ms + sliced reduce "
              f"{max(red):.2f} ms host-timed (sums over the steps)", flush=True)
    union = [e.timing()["union_ms"] / e.timing()["steps"] for e in engines]
    fin = [e.timing()["reduce_ms"] / e.timing()["steps"] for e in engines]
    arcs = [int(g.offsets()[hi]) - int(g.offsets()[lo]) for lo, hi in shard_ranges(g.num_nodes(), G)]
    for s in shards:
        s.shard_detach()
    for s in shards:
        s.close()
    return union, fin, rows, arcs


for relabel in (False, True):
    u, f = single(relabel)
    print(f"single engine relabel={relabel}: union {u:.3f} ms, finish {f:.3f} ms "
          f"(steps 1-2 mean)", flush=True)
for relabel, scatter in ((False, "1"), (True, "1"), (True, "0")):
    u, f, rows, arcs = sharded(relabel, scatter)
    print(f"{G} shards relabel={relabel} est_scatter={scatter}: union per shard max {max(u):.3f} mean "
          f"{sum(u) / len(u):.3f} ms, finish mean {sum(f) / len(f):.3f} ms; "
          f"N(1)={rows[0].sum!r} N(2)={rows[1].sum!r}", flush=True)
    print("   union ms per shard:", " ".join(f"{x:.3f}" for x in u), flush=True)
