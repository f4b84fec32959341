"""Dev aid: one dense step of R-MAT scale k (GPU-generated), for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
g = h.gen_rmat(int(sys.argv[1]), 16, 0.57, 0.19, 0.19, 1, 7, device=0)
e = h.NfEngine(g, h.EngineConfig(bucket_bits=6, seed=42, exact_sum=False))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    e.reset(); e.step()
print("ok")
