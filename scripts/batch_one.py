import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
g = h.gen_rmat(int(sys.argv[1]), 16, 0.57, 0.19, 0.19, 1, 7, device=0)
K = int(sys.argv[2])
runs = h.multirun(g, h.EngineConfig(bucket_bits=6, seed=42), runs=K, batch=K)
print("ok", [r.iterations() for r in runs])
