"""Dev aid: share of arcs whose successor lands in the first H rows after
degree relabelling (descending out-degree), for the propagation-blocking
design (DESIGN 5.6).  python scripts/hot_fraction.py CONFIG"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
cfg = int(sys.argv[1])
t = time.time()
g = bench.make_graph(cfg, device=0 if bench.CONFIGS[cfg]["kind"] == "rmat" else None)
n, a = g.num_nodes(), g.num_arcs()
off = torch.from_numpy(g.offsets().view(np.int64)).cuda()
deg = off[1:] - off[:-1]
order = torch.argsort(-deg, stable=True)
rank = torch.empty(n, dtype=torch.int32, device="cuda")
rank[order] = torch.arange(n, dtype=torch.int32, device="cuda")
indeg = torch.zeros(n, dtype=torch.int64, device="cuda")
succ = g.arcs()
step = 1 << 28
for lo in range(0, a, step):
    s = torch.from_numpy(succ[lo:lo + step].astype(np.int64)).cuda()
    indeg.index_add_(0, rank[s].long(), torch.ones_like(s))
cum = torch.cumsum(indeg, 0).cpu().numpy()
print(f"config {cfg}: n={n} a={a} ({time.time() - t:.1f} s)")
for k in range(14, 30):
    H = 1 << k
    if H > n: break
    print(f"  H=2^{k:2d} rows: {cum[H - 1] / a:.4f} of arcs")
# in-degree of the hottest rows vs out-degree order
print("  zero out-degree rows:", int((deg == 0).sum()))
