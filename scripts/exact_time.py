"""Dev aid: exact N(t) on the GPU vs the reference's all-pairs BFS (16 threads)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
import oracle
for scale in (14, 16):
    g = h.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7)
    h.exact_nf(h.gen_rmat(8, 4))
    t0 = time.perf_counter(); e = h.exact_nf(g); t1 = time.perf_counter()
    line = f"R-MAT {scale} ({g.num_nodes()} nodes, {g.num_arcs()} arcs): GPU {t1 - t0:.3f} s, diameter {e.diameter()}"
    if oracle.have_ref():
        R = oracle.ref()
        rg = R.graph(g.num_nodes(), g.offsets(), g.arcs())
        t0 = time.perf_counter(); want = R.exact_nf(rg); t1 = time.perf_counter()
        line += f", reference BFS {t1 - t0:.3f} s, equal {want == e.values}"
    print(line, flush=True)
