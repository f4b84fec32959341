"""Does a locality order (reverse Cuthill-McKee on the host, scipy) beat
the engine's degree relabelling on DRAM-bound graphs?  Union sweep time of
dense steps 1-2 (CUDA events), same graph renumbered.

  python scripts/order_probe.py rmat|ba SCALE
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
from scipy.sparse.csgraph import reverse_cuthill_mckee  # noqa: E402

import paper_1011_5599_b200 as hanf  # noqa: E402

kind, scale = sys.argv[1], int(sys.argv[2])
t0 = time.time()
if kind == "rmat":
    g = hanf.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
    b = 6
else:
    g = hanf.gen_barabasi_albert(1 << scale, 10, 4, 11)
    b = 5
n, off, arcs = g.num_nodes(), g.offsets(), g.arcs()
print(f"{kind} {scale}: n={n} arcs={len(arcs)} ({time.time() - t0:.1f} s)", flush=True)


def sweep_ms(graph, env):
    for k, v in env.items():
        os.environ[k] = v
    with hanf.NfEngine(graph, hanf.EngineConfig(bucket_bits=b, seed=42, exact_sum=False)) as e:
        e.set_timing(True)
        e.step()
        e.step()
        t = e.timing()
    for k in env:
        del os.environ[k]
    return t["union_ms"] / t["steps"], t["reduce_ms"] / t["steps"]


print("original ids, default (degree relabel):", sweep_ms(g, {}), flush=True)
print("original ids, no relabel:", sweep_ms(g, {"HANF_RELABEL": "0"}), flush=True)
t0 = time.time()
A = sp.csr_matrix((np.ones(len(arcs), dtype=np.int8), arcs.astype(np.int32), off.astype(np.int64)),
                  shape=(n, n))
perm = reverse_cuthill_mckee(A, symmetric_mode=(kind == "ba"))
print(f"RCM {time.time() - t0:.1f} s", flush=True)
inv = np.empty(n, dtype=np.int64)
inv[perm] = np.arange(n)
deg = np.diff(off.astype(np.int64))
new_deg = deg[perm]
new_off = np.zeros(n + 1, dtype=np.uint64)
np.cumsum(new_deg, out=new_off[1:])
src_new = np.repeat(inv[np.arange(n)], deg)  # new id of each arc's source (old order)
dst_new = inv[arcs]
order = np.lexsort((dst_new, src_new))
new_arcs = dst_new[order].astype(np.uint32)
rg = hanf.Graph(n, new_off, new_arcs)
print(f"renumbered ({time.time() - t0:.1f} s)", flush=True)
print("RCM ids, no relabel:", sweep_ms(rg, {"HANF_RELABEL": "0"}), flush=True)
print("RCM ids, segments:", sweep_ms(rg, {"HANF_RELABEL": "0", "HANF_SEGMENTS": "1"}), flush=True)
# reversed RCM = Cuthill-McKee
print("RCM ids, default:", sweep_ms(rg, {}), flush=True)
