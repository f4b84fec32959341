"""Quick GPU probe: parity on a few graphs + rough step timing (dev aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1011_5599_b200 as h

P = oracle.port()
def lockstep(g, steps=40, **cfg):
    pe = P.engine(g.num_nodes(), g.offsets(), g.arcs(), **cfg)
    with h.NfEngine(g, h.EngineConfig(**cfg)) as e:
        assert e.sum_estimates() == pe.sum_estimates(), "N0"
        for t in range(steps):
            r = e.step(); s, m = pe.step()
            ok = (r.sum == s and r.modified == m and np.array_equal(e.counters(), pe.counters()))
            if not ok:
                print("MISMATCH", cfg, t, r, s, m); return False
            if m == 0: break
    print("ok", g.num_nodes(), g.num_arcs(), cfg, t); return True

for b, r in [(6, 0), (7, 0), (5, 0), (4, 0), (4, 6), (5, 6), (6, 7), (4, 7), (8, 0), (5, 8), (9, 0)]:
    lockstep(h.gen_uniform_random(2000, 5, 3), bucket_bits=b, register_bits=r, seed=42)
lockstep(h.gen_rmat(14), bucket_bits=6, seed=42)
lockstep(h.gen_clique_path(40, 10), bucket_bits=7, seed=42)

g = h.gen_rmat(20)
print("rmat20", g.num_arcs())
for b in (6, 7, 5):
    e = h.NfEngine(g, h.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
    ts = []
    for k in range(5):
        e.reset()
        t0 = time.perf_counter(); r = e.step(); ts.append(time.perf_counter() - t0)
    print("b", b, "dense step ms", [round(x * 1e3, 3) for x in ts], "arcs/s %.3e" % (g.num_arcs() / min(ts)))
    e.reset()
    t0 = time.perf_counter(); est = e.run_to_stabilisation(); dt = time.perf_counter() - t0
    print("  full run", est.iterations(), "iters", round(dt * 1e3, 2), "ms", est.modified[:6])
    e.close()
