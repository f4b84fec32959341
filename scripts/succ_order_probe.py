"""Does the order of each node's successors matter to the union sweep?
(Results do not depend on it.)  Lanes of a warp fold trip row i together:
if row i holds every node's most popular successor, lanes of one gather
instruction share L1 lines.  Config 2, dense steps 1-2, CUDA events.

  python scripts/succ_order_probe.py [config]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1011_5599_b200 as hanf  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "2"
if arg.startswith("rmat"):  # e.g. rmat24: a DRAM-bound R-MAT, m = 64
    name, b = arg, 6
    g = hanf.gen_rmat(int(arg[4:]), 16, 0.57, 0.19, 0.19, 1, 7, device=0)
elif arg.startswith("ba"):  # e.g. ba24: Barabasi-Albert 2^24, m = 32
    name, b = arg, 5
    g = hanf.gen_barabasi_albert(1 << int(arg[2:]), 10, 4, 11)
else:
    name, make, b = bench.workload(int(arg))
    g = make()
n, off, arcs = g.num_nodes(), g.offsets(), g.arcs()
deg = np.diff(off.astype(np.int64))
src = np.repeat(np.arange(n, dtype=np.int64), deg)
indeg = np.bincount(arcs, minlength=n)


def sweep_ms(graph, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    with hanf.NfEngine(graph, hanf.EngineConfig(bucket_bits=b, seed=42, exact_sum=False)) as e:
        e.set_timing(True)
        for _ in range(3):
            e.step()
        t = e.timing()
    for k in (env or {}):
        del os.environ[k]
    return round(t["union_ms"] / t["steps"], 4)


def reorder(key):
    o = np.lexsort((key, src))
    return hanf.Graph(n, off.copy(), arcs[o].copy())


print(name, flush=True)
sweep_ms(g)  # (first engine of the process: lazy kernel loading)
print("csr order (ids ascending):", sweep_ms(g), sweep_ms(g, {"HANF_RELABEL": "1"}), flush=True)
print("popular first (in-degree desc):", sweep_ms(reorder(-indeg[arcs])),
      sweep_ms(reorder(-indeg[arcs]), {"HANF_RELABEL": "1"}), flush=True)
rng = np.random.default_rng(1)
print("random order:", sweep_ms(reorder(rng.random(len(arcs)))), flush=True)
