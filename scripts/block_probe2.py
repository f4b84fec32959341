"""Dev aid (probe for a source-blocked pass, part 2): upper bound of the
blocked pass.  The arcs (source rank < 2^S, successor rank >= 2^T) of config
C become (successor segment, source) items; the items are the only nodes
with arcs of a stand-in graph in rank space (item k = node n + k), grouped
segment-major (HANF_SEGMENTS=1), and its dense sweep is timed.
    python scripts/block_probe2.py CONFIG S_LOG2 T_LOG2 SEG_LOG2 GROUP_SHIFT"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1011_5599_b200 as h

cfg = int(sys.argv[1])
S, T, SEG, GSH = (int(x) for x in sys.argv[2:6])
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
del order, deg
keys, vals = [], []
step = 1 << 27
for lo in range(0, a, step):
    hi = min(a, lo + step)
    idx = torch.arange(lo, hi, dtype=torch.int64, device="cuda")
    src = torch.searchsorted(off, idx, right=True) - 1
    del idx
    dst = torch.from_numpy(succ_h[lo:hi].view(np.int32)).cuda()
    rs = rank[src]
    rd = rank[dst.long() & 0xffffffff]
    blk = (rs < (1 << S)) & (rd >= (1 << T))
    keys.append(((rd[blk].long() >> SEG) << 24) | rs[blk].long())
    vals.append(rd[blk])
    del src, dst, rs, rd, blk
del off, rank
key = torch.cat(keys); del keys
val = torch.cat(vals); del vals
key, perm = torch.sort(key)
val = val[perm]; del perm
_, counts = torch.unique_consecutive(key, return_counts=True)
del key
items = counts.numel()
print(f"blocked arcs {val.numel()}, items {items}, max item {int(counts.max())}", flush=True)
N = n + items
offs = torch.zeros(N + 1, dtype=torch.int64, device="cuda")
offs[n + 1:] = torch.cumsum(counts, 0)
g2 = h.Graph(N, offs.cpu().numpy().view(np.uint64), val.cpu().numpy().view(np.uint32))
del offs, val, counts, g
torch.cuda.empty_cache()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
os.environ.update(HANF_RELABEL="0", HANF_SEGMENTS="1", HANF_SEG_SHIFT=str(GSH), HANF_LAYOUT="packed")
e = h.NfEngine(g2, h.EngineConfig(bucket_bits=c["b"], seed=42, exact_sum=False))
e.reset(); e.step()
e.set_timing(True)
for _ in range(4):
    e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
t = e.timing()
print(f"config {cfg} items S=2^{S} T=2^{T} seg=2^{SEG} group=2^{GSH}: union "
      f"{t['union_ms'] / t['steps']:.3f} ms for {g2.num_arcs()} arcs", flush=True)
e.close()
