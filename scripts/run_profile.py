"""Per-iteration device time of one whole run (HANF timing events):
python scripts/run_profile.py CONFIG [--summary]"""
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1011_5599_b200 as hanf  # noqa: E402

cfg_id = int(sys.argv[1])
name, make, b = bench.workload(cfg_id)
t0 = time.time()
g = make()
n = g.num_nodes()
print(f"{name}: n={n} arcs={g.num_arcs()} generated in {time.time() - t0:.1f} s", flush=True)
t0 = time.time()
e = hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=b, seed=42))
print(f"create {time.time() - t0:.2f} s", flush=True)
t0 = time.time()
est = e.run_to_stabilisation()
print(f"run_to_stabilisation {time.time() - t0:.3f} s, T={est.iterations()}", flush=True)
e.reset()
rows = []
prev = n
t0 = time.time()
while True:
    e.set_timing(True)
    rep = e.step()
    t = e.timing()
    rows.append((len(rows) + 1, rep.modified, prev, t["union_ms"], t["reduce_ms"] + t["estimate_ms"]))
    prev = rep.modified
    if rep.modified == 0:
        break
wall = time.time() - t0
print(f"timed replay: {len(rows)} steps, wall {wall:.3f} s, device sweep "
      f"{sum(r[3] for r in rows) / 1e3:.3f} s, finish {sum(r[4] for r in rows) / 1e3:.3f} s")
# buckets by the previous step's modified count (what picks the step mode)
buckets = defaultdict(lambda: [0, 0.0, 0.0])
for t, mod, p, u, f in rows:
    k = "dense (prev >= n/2)" if 2 * p >= n else (
        "prev >= n/128" if 128 * p >= n else
        "prev >= n/4096" if 4096 * p >= n else "prev < n/4096")
    buckets[k][0] += 1
    buckets[k][1] += u
    buckets[k][2] += f
for k, (c, u, f) in buckets.items():
    print(f"  {k:22s} steps {c:6d} sweep {u:9.2f} ms ({u / c:.3f}/step) finish {f:8.2f} ms")
if "--summary" not in sys.argv:
    for r in rows[:12] + rows[-5:]:
        print("  t=%d modified=%d prev=%d sweep=%.3f finish=%.3f" % r)
