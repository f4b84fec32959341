"""Dev aid: config C dense iteration with source-blocked sweeps (HANF_BLOCK=1
at create) under env variants, against the plain sweep.
    python scripts/block_time.py CONFIG "ENV1;ENV2;..."   (ENV = K=V,K=V)"""
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
    t0 = time.time()
    e = h.NfEngine(g, h.EngineConfig(bucket_bits=c["b"], seed=42, exact_sum=False))
    torch.cuda.synchronize()
    t_create = time.time() - t0
    for k, v in old.items():
        if v is None: os.environ.pop(k)
        else: os.environ[k] = v
    e.reset(); r1 = e.step()
    e.set_timing(True)
    for _ in range(4):
        e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
    t = e.timing()
    e.set_timing(False)
    e.reset()
    t0 = time.time()
    est = e.run_to_stabilisation()
    t_run = time.time() - t0
    print(f"config {cfg} [{spec or 'default'}]: create {t_create:.3f} s, block {e.block_stats()}, "
          f"union {t['union_ms'] / t['steps']:.3f} ms, N(1)={r1.sum!r} mod={r1.modified}, "
          f"run {t_run:.3f} s, {len(est.values)} values, last {est.values[-1]!r}", flush=True)
    e.close()
