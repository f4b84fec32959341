"""Dev aid: one dense step of a config with a given variant (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1011_5599_b200 as h
name, make, b = bench.workload(int(sys.argv[1]))
g = make()
e = h.NfEngine(g, h.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    e.reset(); e.step()
print("ok")
