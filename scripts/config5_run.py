"""Dev aid: one whole estimate_nf on BASELINE config 5 (R-MAT 28, 4.26 B arcs)."""
import os, sys, time
os.environ.setdefault("HANF_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as h
t0 = time.perf_counter(); g = h.gen_rmat(28, 16, 0.57, 0.19, 0.19, 1, 7, device=0); t1 = time.perf_counter()
print(f"generate (GPU): {t1 - t0:.1f} s, {g.num_nodes()} nodes, {g.num_arcs()} arcs", flush=True)
t0 = time.perf_counter(); g.pin(); t1 = time.perf_counter()
print(f"pin: {t1 - t0:.1f} s", flush=True)
cfg = h.EngineConfig(bucket_bits=6, seed=42)
t0 = time.perf_counter(); e = h.NfEngine(g, cfg); t1 = time.perf_counter()
print(f"create: {t1 - t0:.2f} s", flush=True)
ts = []
while True:
    a = time.perf_counter(); r = e.step(); b = time.perf_counter()
    ts.append((b - a, r.modified, r.sum))
    print(f"  step {len(ts)}: {1e3 * (b - a):8.1f} ms  modified {r.modified:>10}  N {r.sum:.6e}", flush=True)
    if r.modified == 0 or len(ts) > 60:
        break
tot = sum(t for t, _, _ in ts)
print(f"run: {tot:.2f} s for {len(ts)} steps, {g.num_arcs() * len(ts) / tot / 1e9:.1f} G arcs/s", flush=True)
e.close()
