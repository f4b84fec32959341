"""Dev aid: one estimate_nf on a config (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1011_5599_b200 as h
name, make, b = bench.workload(int(sys.argv[1]))
g = make()
est = h.estimate_nf(g, h.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
print("iterations", est.iterations())
