"""Dev aid: multirun throughput: re-seeded engine (batch=1) vs batched engines."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
name = sys.argv[1] if len(sys.argv) > 1 else "rmat20"
scale = int(name[4:])
g = h.gen_rmat(scale, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
pg = h.Graph(g.num_nodes(), g.offsets().copy(), g.arcs().copy()).pin()
cfg = h.EngineConfig(bucket_bits=6, seed=42)
R = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ref = None
for batch in (1, 2, 4, 8):
    h.multirun(pg, cfg, runs=batch, batch=batch)  # warm
    t0 = time.perf_counter(); runs = h.multirun(pg, cfg, runs=R, batch=batch); t1 = time.perf_counter()
    its = sum(r.iterations() + 1 for r in runs)
    if ref is None:
        ref = runs
    same = all(a.values == b.values for a, b in zip(runs, ref))
    print(f"{name} R={R} batch={batch}: {1e3*(t1-t0):8.1f} ms  {g.num_arcs()*its/(t1-t0)/1e9:6.1f} G arc-runs/s  identical {same}", flush=True)
