"""Dev aid: does relabelling nodes by in-degree (hot counters packed
together) speed up the union sweep on DRAM-bound graphs?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1011_5599_b200 as h


def union_ms(g, b):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e = h.NfEngine(g, h.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
    e.reset(); e.step()
    e.set_timing(True)
    for _ in range(3):
        e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
    t = e.timing(); e.close()
    k = t["steps"]
    print(f"    (union {t['union_ms'] / k:.3f} + estimate {t['estimate_ms'] / k:.3f} + finish {t['reduce_ms'] / k:.3f} ms)", flush=True)
    return t["union_ms"] / k


def relabel(g, key):
    dev = torch.device("cuda")
    n = g.num_nodes()
    off = torch.from_numpy(g.offsets().view(np.int64)).to(dev)
    arcs = torch.from_numpy(g.arcs().view(np.int32)).to(dev).long()
    deg = off[1:] - off[:-1]
    indeg = torch.bincount(arcs, minlength=n)
    score = {"indeg": indeg, "out": deg}.get(key, indeg + deg)
    order = torch.argsort(-score, stable=True)          # new id -> old id
    perm = torch.empty_like(order); perm[order] = torch.arange(n, device=dev)
    ndeg = deg[order]
    noff = torch.zeros(n + 1, dtype=torch.long, device=dev); noff[1:] = torch.cumsum(ndeg, 0)
    start = torch.repeat_interleave(off[:-1][order] - noff[:-1], ndeg)
    src_idx = torch.arange(arcs.numel(), device=dev) + start
    narcs = perm[arcs[src_idx]].int()
    out = h.Graph(n, noff.cpu().numpy().view(np.uint64), narcs.cpu().numpy().view(np.uint32))
    del off, arcs, deg, indeg, order, perm, ndeg, noff, start, src_idx, narcs
    torch.cuda.empty_cache()
    return out


for cfg in sys.argv[1].split(","):
    if cfg == "rmat26":
        name, make, b = "R-MAT 26 (ef 16, ids permuted)", (lambda: h.gen_rmat(26, 16, 0.57, 0.19, 0.19, 1, 7)), 6
    else:
        name, make, b = bench.workload(int(cfg))
    t0 = time.time(); g = make(); print(name, f"gen {time.time() - t0:.1f} s, arcs {g.num_arcs()}", flush=True)
    a = g.num_arcs()
    os.environ["HANF_RELABEL"] = "1"
    u2 = union_ms(g, b)
    print(f"  engine relabel union {u2:8.3f} ms  {a / u2 / 1e6:6.1f} G arcs/s", flush=True)
    os.environ["HANF_RELABEL"] = "0"
    for key in ("total", "out"):
        t0 = time.time(); r = relabel(g, key); t1 = time.time()
        u1 = union_ms(r, b)
        print(f"  by {key:6s}     union {u1:8.3f} ms  {a / u1 / 1e6:6.1f} G arcs/s  (relabel {t1 - t0:.1f} s)", flush=True)
        del r
    del g
