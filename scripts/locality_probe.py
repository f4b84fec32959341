"""Dev aid: does the union sweep exploit config 3's id locality?  Compare the
graph as generated (local ids), randomly permuted ids, and ids sorted by
(out-degree, id) - the task order - applied as a relabelling."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1011_5599_b200 as h
os.environ["HANF_RELABEL"] = "0"


def union_ms(g, b):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e = h.NfEngine(g, h.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
    e.reset(); e.step()
    e.set_timing(True)
    for _ in range(3):
        e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
    t = e.timing(); e.close()
    return t["union_ms"] / t["steps"]


def permuted(g, order):
    dev = torch.device("cuda")
    n = g.num_nodes()
    off = torch.from_numpy(g.offsets().view(np.int64)).to(dev)
    arcs = torch.from_numpy(g.arcs().view(np.int32)).to(dev).long()
    order = order.to(dev)
    perm = torch.empty_like(order); perm[order] = torch.arange(n, device=dev)
    deg = off[1:] - off[:-1]
    ndeg = deg[order]
    noff = torch.zeros(n + 1, dtype=torch.long, device=dev); noff[1:] = torch.cumsum(ndeg, 0)
    start = torch.repeat_interleave(off[:-1][order] - noff[:-1], ndeg)
    narcs = perm[arcs[torch.arange(arcs.numel(), device=dev) + start]].int()
    return h.Graph(n, noff.cpu().numpy().view(np.uint64), narcs.cpu().numpy().view(np.uint32))


name, make, b = bench.workload(3)
g = make()
print(name, flush=True)
print(f"  local ids      union {union_ms(g, b):.3f} ms", flush=True)
n = g.num_nodes()
gen = torch.Generator().manual_seed(5)
rnd = permuted(g, torch.randperm(n, generator=gen))
print(f"  random ids     union {union_ms(rnd, b):.3f} ms", flush=True)
del rnd
deg = torch.from_numpy((g.offsets()[1:] - g.offsets()[:-1]).astype(np.int64))
bydeg = permuted(g, torch.argsort(-deg, stable=True))
print(f"  (deg, id) ids  union {union_ms(bydeg, b):.3f} ms", flush=True)
