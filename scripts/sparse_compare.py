"""Dev aid: per-iteration step time, dense sweep with skipping vs the
opt-in worklist step (HANF_SPARSE=1), on BASELINE configs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401  (initialises CUDA the same way bench.py does)
import bench
import paper_1011_5599_b200 as h

for cfgno in [int(c) for c in sys.argv[1].split(",")]:
    name, make, b = bench.workload(cfgno)
    g = make()
    print(name, flush=True)
    rows = {}
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1"]
    for mode in modes:
        if mode == "default":
            os.environ.pop("HANF_SPARSE", None)
        else:
            os.environ["HANF_SPARSE"] = mode
        for rep in range(2):  # second run: graphs captured, transpose built
            e = h.NfEngine(g, h.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
            if rep == 1:
                e.run_to_stabilisation(); e.reset()
            times = []
            while True:
                t0 = time.perf_counter(); r = e.step(); t1 = time.perf_counter()
                times.append((1e3 * (t1 - t0), r.modified))
                if r.modified == 0:
                    break
            e.close()
        rows[mode] = times
    pairs = list(zip(rows[modes[0]], rows[modes[1]]))
    print("columns:", modes)
    if len(pairs) <= 40:
        print(f"{'t':>3} {'modified':>10} {'dense+skip ms':>14} {'worklist ms':>12}")
        for t, ((a, m), (c, _)) in enumerate(pairs, 1):
            print(f"{t:>3} {m:>10} {a:>14.3f} {c:>12.3f}")
    else:  # bucket iterations by log2(modified)
        import math
        buckets = {}
        for (a, m), (c, _) in pairs:
            k = int(math.log2(m + 1))
            n_, sa, sc = buckets.get(k, (0, 0.0, 0.0))
            buckets[k] = (n_ + 1, sa + a, sc + c)
        print(f"{'log2 mod':>8} {'iters':>6} {'dense+skip ms':>14} {'worklist ms':>12}")
        for k in sorted(buckets):
            n_, sa, sc = buckets[k]
            print(f"{k:>8} {n_:>6} {sa / n_:>14.3f} {sc / n_:>12.3f}")
    print(f"total {sum(x for x, _ in rows[modes[0]]):.3f} ms vs {sum(x for x, _ in rows[modes[1]]):.3f} ms", flush=True)
