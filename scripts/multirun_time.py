"""Dev aid: multirun (one engine, re-seeded) vs independent estimate_nf calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
g = h.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7)
pg = h.Graph(g.num_nodes(), g.offsets().copy(), g.arcs().copy()).pin()
cfg = h.EngineConfig(bucket_bits=6, seed=42)
h.estimate_nf(pg, cfg)
for R in (10, 100):
    t0 = time.perf_counter(); runs = h.multirun(pg, cfg, runs=R); t1 = time.perf_counter()
    t2 = time.perf_counter(); ind = [h.estimate_nf(pg, h.EngineConfig(bucket_bits=6, seed=42 + i)) for i in range(R)]; t3 = time.perf_counter()
    same = all(a.values == b.values for a, b in zip(runs, ind))
    its = sum(r.iterations() + 1 for r in runs)
    print(f"R={R}: multirun {1e3*(t1-t0):.1f} ms ({g.num_arcs()*its/(t1-t0)/1e9:.1f} G arcs/s), "
          f"independent {1e3*(t3-t2):.1f} ms, identical {same}", flush=True)
    rep = h.aggregate_runs(runs)
    print("  spid mean/sd", rep.spid_mean if hasattr(rep, 'spid_mean') else rep)
