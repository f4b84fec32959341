"""Dev aid (probe for a source-blocked pass): dense-sweep time of config C
with the arcs (source rank < S, successor rank >= T) removed, and how those
arcs would group into (successor segment, source) items.
    python scripts/block_probe.py CONFIG "S_LOG2,T_LOG2,SEG_LOG2;..." """
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1011_5599_b200 as h

cfg = int(sys.argv[1])
c = bench.CONFIGS[cfg]
g = bench.make_graph(cfg, device=0 if c["kind"] == "rmat" else None)
n, a = g.num_nodes(), g.num_arcs()
off_h = g.offsets()
succ_h = g.arcs()
off = torch.from_numpy(off_h.view(np.int64)).cuda()
deg = off[1:] - off[:-1]
order = torch.argsort(-deg, stable=True)
rank = torch.empty(n, dtype=torch.int32, device="cuda")
rank[order] = torch.arange(n, dtype=torch.int32, device="cuda")
del order
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def time_engine(graph, label):
    e = h.NfEngine(graph, h.EngineConfig(bucket_bits=c["b"], seed=42, exact_sum=False))
    e.reset(); e.step()
    e.set_timing(True)
    for _ in range(4):
        e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
    t = e.timing()
    e.set_timing(False)
    print(f"config {cfg} [{label}]: arcs {graph.num_arcs()}  union "
          f"{t['union_ms'] / t['steps']:.3f} ms", flush=True)
    e.close()


time_engine(g, "full graph")
step = 1 << 27
for spec in sys.argv[2].split(";"):
    S, T, SEG = (int(x) for x in spec.split(","))
    kept_chunks, counts = [], torch.zeros(n, dtype=torch.int64, device="cuda")
    blocked = 0
    items = 0
    for lo in range(0, a, step):
        hi = min(a, lo + step)
        idx = torch.arange(lo, hi, dtype=torch.int64, device="cuda")
        src = torch.searchsorted(off, idx, right=True) - 1
        del idx
        dst = torch.from_numpy(succ_h[lo:hi].view(np.int32)).cuda()
        rs = rank[src]
        rd = rank[dst.long() & 0xffffffff]
        blk = (rs < (1 << S)) & (rd >= (1 << T))
        blocked += int(blk.sum())
        # (segment, source) items among the blocked arcs of this chunk
        key = (rs[blk].long() << 20) | (rd[blk].long() >> SEG)
        items += int(torch.unique(key).numel())
        del key, rs, rd
        keep = ~blk
        counts.index_add_(0, src[keep], torch.ones(int(keep.sum()), dtype=torch.int64, device="cuda"))
        kept_chunks.append(dst[keep].cpu().numpy().view(np.uint32))
        del src, dst, blk, keep
    new_off = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    new_off[1:] = torch.cumsum(counts, 0)
    arcs2 = np.concatenate(kept_chunks)
    del kept_chunks
    g2 = h.Graph(n, new_off.cpu().numpy().view(np.uint64), arcs2)
    print(f"  S=2^{S} T=2^{T} seg=2^{SEG}: blocked {blocked} arcs ({blocked / a:.3f}), "
          f"{items} (segment, source) items ({blocked / max(1, items):.2f} arcs each), "
          f"{(n - (1 << T)) >> SEG} segments", flush=True)
    time_engine(g2, f"without blocked arcs S=2^{S} T=2^{T}")
    del g2, arcs2
