"""Dev aid: per-step sweep/finish times of one whole run (bench.run_profile)
plus the wall time of a warm estimate_nf, for a BASELINE config.
    python scripts/run_profile.py CONFIG"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1011_5599_b200 as h
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = bench.CONFIGS[cfg_id]
g = bench.make_graph(cfg_id, device=0 if c["kind"] == "rmat" else None)
e = h.NfEngine(g, h.EngineConfig(bucket_bits=c["b"], seed=bench.HLL_SEED, exact_sum=False))
for row in bench.run_profile(e, g.num_nodes()):
    print(json.dumps(row))
e.close()
g.pin()
cfg = h.EngineConfig(bucket_bits=c["b"], seed=bench.HLL_SEED)
h.estimate_nf(g, cfg)
for _ in range(2):
    t0 = time.perf_counter()
    est = h.estimate_nf(g, cfg)
    print(f"estimate_nf {1e3 * (time.perf_counter() - t0):.1f} ms, {est.iterations() + 1} steps")
