"""Dev aid: SM clocks and throttle reasons during back-to-back config 5 runs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_1011_5599_b200 as h
g = bench.make_graph(5, device=0)
e = h.NfEngine(g, h.EngineConfig(bucket_bits=6, seed=bench.HLL_SEED, exact_sum=False))
e.run_to_stabilisation()
with bench.ClockSampler(0) as clocks:
    for _ in range(4):
        e.reset()
        e.run_to_stabilisation()
print(clocks.summary())
for row in bench.run_profile(e, g.num_nodes())[:6]:
    print(row)
e.close()
