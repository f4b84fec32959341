"""Dev aid: union-sweep time of config 5's dense iteration 1 when only the
gathers of rows in [lo, hi) are performed (HANF_DBG_RANGE, timing only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1011_5599_b200 as h
cfg = int(sys.argv[1])
c = bench.CONFIGS[cfg]
g = bench.make_graph(cfg, device=0 if c["kind"] == "rmat" else None)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e = h.NfEngine(g, h.EngineConfig(bucket_bits=c["b"], seed=42, exact_sum=False))
for spec in sys.argv[2].split(";"):
    if spec:
        os.environ["HANF_DBG_RANGE"] = spec
    else:
        os.environ.pop("HANF_DBG_RANGE", None)
    e.reset(); e.step()
    e.set_timing(True)
    for _ in range(3):
        e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
    t = e.timing()
    e.set_timing(False)
    print(f"config {cfg} [{spec or 'all'}]: union {t['union_ms'] / t['steps']:.3f} ms", flush=True)
e.close()
