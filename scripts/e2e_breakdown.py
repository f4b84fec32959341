"""Where the time of a one-shot estimate_nf goes (config 2, page-locked CSR):
create vs run, and the device time of each step (CUDA events around the
step's kernels, an ungraphed replay of the same run)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1011_5599_b200 as hanf  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
name, make, b = bench.workload(cfg_id)
g0 = make()
g = hanf.Graph(g0.num_nodes(), g0.offsets().copy(), g0.arcs().copy()).pin()
cfg = hanf.EngineConfig(bucket_bits=b, seed=42)
hanf.estimate_nf(g, cfg)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    est = hanf.estimate_nf(g, cfg)
    t1 = time.perf_counter()
    e = hanf.NfEngine(g, cfg)
    t2 = time.perf_counter()
    e.run_to_stabilisation()
    t3 = time.perf_counter()
    e.close()
    t4 = time.perf_counter()
    print(f"estimate_nf {1e3 * (t1 - t0):.3f} ms | create {1e3 * (t2 - t1):.3f} run "
          f"{1e3 * (t3 - t2):.3f} destroy {1e3 * (t4 - t3):.3f} ms; T={est.iterations()}", flush=True)
with hanf.NfEngine(g, cfg) as e:
    e.set_timing(True)
    walls = []
    while True:
        before = e.timing()
        t0 = time.perf_counter()
        rep = e.step()
        walls.append(1e3 * (time.perf_counter() - t0))
        after = e.timing()
        print(f"step {len(walls)}: modified {rep.modified:9d} wall {walls[-1]:.3f} ms, union "
              f"{after['union_ms'] - before['union_ms']:.3f} est "
              f"{after['estimate_ms'] - before['estimate_ms']:.3f} finish "
              f"{after['reduce_ms'] - before['reduce_ms']:.3f} ms", flush=True)
        if rep.modified == 0:
            break
