"""Dev aid: per-run wall of a re-seeded config 5 engine (where a multi-run's time goes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
g = h.gen_rmat(28, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
g.pin()
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = h.EngineConfig(bucket_bits=6, seed=42, expected_runs=int(os.environ.get("RUNS_HINT", "0")))
h.estimate_nf(g, cfg)
t0 = time.perf_counter()
e = h.NfEngine(g, cfg)
print(f"create {1e3 * (time.perf_counter() - t0):.0f} ms, block {e.block_stats()}", flush=True)
for i in range(runs):
    t0 = time.perf_counter()
    if i:
        e.reseed(42 + i)
    t1 = time.perf_counter()
    est = e.run_to_stabilisation()
    t2 = time.perf_counter()
    print(f"run {i}: reseed {1e3 * (t1 - t0):.0f} ms, run {1e3 * (t2 - t1):.0f} ms "
          f"({est.iterations() + 1} steps), block {e.block_stats()[0]}", flush=True)
e.close()
