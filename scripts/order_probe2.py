"""Dev aid: do locality orders beat the engine's degree relabelling at
scale (R-MAT 26, DRAM-resident counters)?  Dense iteration 1 union sweep
(CUDA events, L2 flushed), the same graph renumbered on the GPU by
  - RCM (scipy, directed structure),
  - BFS over in-arcs from the max-in-degree node (predecessors of a node
    become id neighbours), unreached nodes appended,
  - the degree order's hot prefix (2^20 rows) followed by the RCM order,
each fed with HANF_RELABEL=0, with and without segmented tasks.
    python scripts/order_probe2.py SCALE"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee, breadth_first_order
import torch
import paper_1011_5599_b200 as hanf

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
g = hanf.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
n, off, arcs = g.num_nodes(), g.offsets(), g.arcs()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print(f"R-MAT {scale}: n={n} arcs={len(arcs)}", flush=True)


def sweep_ms(graph, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    with hanf.NfEngine(graph, hanf.EngineConfig(bucket_bits=6, seed=42, exact_sum=False)) as e:
        for k, v in old.items():
            if v is None: os.environ.pop(k)
            else: os.environ[k] = v
        e.reset(); e.step()
        e.set_timing(True)
        for _ in range(3):
            e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
        t = e.timing()
    return round(t["union_ms"] / t["steps"], 3)


def renumber(perm):
    """Graph with node perm[i] renamed i (rows moved, successors mapped), on the GPU."""
    d = torch.device("cuda")
    offt = torch.from_numpy(off.astype(np.int64)).to(d)
    p = torch.from_numpy(perm.astype(np.int64)).to(d)
    inv = torch.empty_like(p); inv[p] = torch.arange(n, device=d)
    deg = offt[1:] - offt[:-1]
    nd = deg[p]
    noff = torch.zeros(n + 1, dtype=torch.int64, device=d); noff[1:] = torch.cumsum(nd, 0)
    rows = torch.repeat_interleave(torch.arange(n, device=d), nd)
    src = offt[p][rows] + torch.arange(len(arcs), device=d) - noff[rows]
    del rows
    a = torch.from_numpy(arcs.astype(np.int64)).to(d)
    na = inv[a[src]].to(torch.int32)
    del a, src
    out = hanf.Graph(n, noff.cpu().numpy().astype(np.uint64), na.cpu().numpy().view(np.uint32))
    torch.cuda.empty_cache()
    return out


res = {"degree relabel (default)": sweep_ms(g, {})}
print(res, flush=True)
A = sp.csr_matrix((np.ones(len(arcs), dtype=np.int8), arcs.astype(np.int32), off.astype(np.int64)),
                  shape=(n, n))
t0 = time.time()
rcm = reverse_cuthill_mckee(A, symmetric_mode=False)
print(f"rcm {time.time() - t0:.1f} s", flush=True)
rg = renumber(rcm)
res["rcm"] = sweep_ms(rg, {"HANF_RELABEL": "0", "HANF_SEGMENTS": "0"})
res["rcm + segments"] = sweep_ms(rg, {"HANF_RELABEL": "0", "HANF_SEGMENTS": "1"})
print(res, flush=True)
del rg
t0 = time.time()
AT = A.T.tocsr()
indeg = np.diff(AT.indptr)
start = int(np.argmax(indeg))
bfs = breadth_first_order(AT, start, directed=True, return_predecessors=False)
seen = np.zeros(n, dtype=bool); seen[bfs] = True
order = np.concatenate([bfs, np.flatnonzero(~seen)])
print(f"in-arc bfs {time.time() - t0:.1f} s ({len(bfs)} reached)", flush=True)
bg = renumber(order)
res["in-bfs"] = sweep_ms(bg, {"HANF_RELABEL": "0", "HANF_SEGMENTS": "0"})
res["in-bfs + segments"] = sweep_ms(bg, {"HANF_RELABEL": "0", "HANF_SEGMENTS": "1"})
print(res, flush=True)
del bg
deg = np.diff(off.astype(np.int64))
hot = np.argsort(-deg, kind="stable")[:1 << 20]
is_hot = np.zeros(n, dtype=bool); is_hot[hot] = True
hyb = np.concatenate([hot, rcm[~is_hot[rcm]]])
hg = renumber(hyb)
res["hot prefix + rcm + segments"] = sweep_ms(hg, {"HANF_RELABEL": "0", "HANF_SEGMENTS": "1"})
res["hot prefix + rcm"] = sweep_ms(hg, {"HANF_RELABEL": "0", "HANF_SEGMENTS": "0"})
print(res, flush=True)
