"""Dev aid: host vs GPU graph construction wall time (configs 2 and 5 R-MAT)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1011_5599_b200 as h
h.gen_rmat(10, 16, device=0)  # context + module load
for scale, host in [(20, True), (24, True), (26, False), (28, False)]:
    t0 = time.perf_counter(); g = h.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7, device=0); t1 = time.perf_counter()
    line = f"R-MAT {scale}: GPU {t1 - t0:7.2f} s ({g.num_arcs()} arcs)"
    if host:
        t0 = time.perf_counter(); r = h.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7); t1 = time.perf_counter()
        line += f", host {t1 - t0:7.2f} s, equal {np.array_equal(r.arcs(), g.arcs()) and np.array_equal(r.offsets(), g.offsets())}"
        del r
    print(line, flush=True)
    del g
