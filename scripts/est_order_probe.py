import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, bench
import paper_1011_5599_b200 as h
g = bench.make_graph(5, device=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e = h.NfEngine(g, h.EngineConfig(bucket_bits=6, seed=42, exact_sum=False))
e.reset(); e.step()
e.set_timing(True)
for _ in range(4):
    e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
t = e.timing()
print(os.environ.get("HANF_EST_ORIG"), {k: (v / t["steps"] if k.endswith("ms") else v) for k, v in t.items()})
