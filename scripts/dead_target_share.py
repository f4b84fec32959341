"""Dev aid: share of arcs whose successor has out-degree 0 (a counter that
never changes after seeding), per BASELINE config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
for c in (int(x) for x in sys.argv[1:] or ["5"]):
    g = bench.make_graph(c, device=0 if bench.CONFIGS[c]["kind"] == "rmat" else None)
    off = torch.from_numpy(g.offsets().astype(np.int64)).cuda()
    dead = (off[1:] - off[:-1]) == 0
    arcs = torch.from_numpy(g.arcs().view(np.int32)).cuda().long()
    share = dead[arcs].float().mean().item()
    print(f"config {c}: nodes {g.num_nodes()}, out-degree 0: {dead.float().mean().item():.3f}, "
          f"arcs into them: {share:.3f}")
