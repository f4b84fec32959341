"""Dev aid: where does estimate_nf's wall time go (config 2)?"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1011_5599_b200 as h
g = h.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7)
torch.cuda.init()
cfg = h.EngineConfig(bucket_bits=6, seed=42)
for k in range(3):
    t0 = time.perf_counter(); e = h.NfEngine(g, cfg); t1 = time.perf_counter()
    est = e.run_to_stabilisation(); t2 = time.perf_counter(); e.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  run {1e3*(t2-t1):.1f} ms ({est.iterations()} it)  destroy {1e3*(t3-t2):.1f} ms")
cfg2 = h.EngineConfig(bucket_bits=6, seed=42, exact_sum=False)
e = h.NfEngine(g, cfg2)
t1 = time.perf_counter(); est = e.run_to_stabilisation(); t2 = time.perf_counter()
print(f"device-sum run {1e3*(t2-t1):.1f} ms")
