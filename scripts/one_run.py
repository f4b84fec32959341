"""Dev aid: one run to stabilisation of a BASELINE config (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1011_5599_b200 as h
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = bench.CONFIGS[cfg_id]
g = bench.make_graph(cfg_id, device=0 if c["kind"] == "rmat" else None)
with h.NfEngine(g, h.EngineConfig(bucket_bits=c["b"], seed=bench.HLL_SEED, exact_sum=False)) as e:
    est = e.run_to_stabilisation()
print(est.iterations())
