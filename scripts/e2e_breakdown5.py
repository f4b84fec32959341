"""Dev aid: phase breakdown of a warm estimate_nf on config 5 (HANF_PROFILE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
g = h.gen_rmat(28, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
g.pin()
cfg = h.EngineConfig(bucket_bits=6, seed=42)
h.estimate_nf(g, cfg)
os.environ.setdefault("HANF_PROFILE", "0")
for _ in range(2):
    t0 = time.perf_counter()
    e = h.NfEngine(g, cfg)
    t1 = time.perf_counter()
    est = e.run_to_stabilisation()
    t2 = time.perf_counter()
    e.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms ({est.iterations()+1} steps)  destroy {1e3*(t3-t2):.1f} ms", flush=True)
