"""Dev aid: union-sweep time of a dense iteration 1 under engine env
variants (HANF_LAYOUT / HANF_SLOTS_HOT ...), one graph.
    python scripts/policy_sweep.py CONFIG "ENV1;ENV2;..."   (ENV = K=V,K=V)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1011_5599_b200 as h
cfg = int(sys.argv[1])
c = bench.CONFIGS[cfg]
g = bench.make_graph(cfg, device=0 if c["kind"] == "rmat" else None)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for spec in sys.argv[2].split(";"):
    env = dict(kv.split("=") for kv in spec.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    e = h.NfEngine(g, h.EngineConfig(bucket_bits=c["b"], seed=42, exact_sum=False))
    for k, v in old.items():
        if v is None: os.environ.pop(k)
        else: os.environ[k] = v
    e.reset(); e.step()
    e.set_timing(True)
    for _ in range(4):
        e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
    t = e.timing()
    e.set_timing(False)
    print(f"config {cfg} [{spec or 'default'}]: union {t['union_ms'] / t['steps']:.3f} ms", flush=True)
    e.close()
