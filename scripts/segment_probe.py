"""Which node segments hold changed counters in the middle of a config-3
run?  Reads the counters back around sampled steps (slow: 1.3 GB each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1011_5599_b200 as hanf  # noqa: E402

name, make, b = bench.workload(3)
g = make()
n = g.num_nodes()
off = g.offsets()
e = hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=b, seed=42))
W = e.params().words
samples = {150, 400, 800, 1200, 1600, 2000, 2400}
prev = e.counters().reshape(n, W)
t = 0
while True:
    rep = e.step()
    t += 1
    if t in samples or rep.modified == 0:
        cur = e.counters().reshape(n, W)
        changed = np.any(cur != prev, axis=1)
        segs = changed.reshape(-1, 1 << 16).any(axis=1)
        idx = np.nonzero(changed)[0]
        print(f"t={t} modified={rep.modified} ({rep.modified / n:.4f}) segments with a change "
              f"{segs.sum()}/256; changed ids: min {idx.min() if len(idx) else -1} max "
              f"{idx.max() if len(idx) else -1}; 64-node blocks with a change "
              f"{changed.reshape(-1, 64).any(axis=1).mean():.4f}", flush=True)
        prev = cur
    elif t + 1 in samples:
        prev = e.counters().reshape(n, W)
    if rep.modified == 0:
        break
