"""Dev aid: estimate_nf phases on config 2 from pinned host CSR (HANF_PROFILE=1)."""
import os, sys, time
os.environ["HANF_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1011_5599_b200 as h
g = h.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7)
pg = h.Graph(g.num_nodes(), g.offsets().copy(), g.arcs().copy()).pin()
torch.cuda.init()
cfg = h.EngineConfig(bucket_bits=6, seed=42, exact_sum=False)
for k in range(4):
    t0 = time.perf_counter(); e = h.NfEngine(pg, cfg); t1 = time.perf_counter()
    est = e.run_to_stabilisation(); t2 = time.perf_counter(); e.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.3f} ms  run {1e3*(t2-t1):.3f} ms ({est.iterations()} it)  close {1e3*(t3-t2):.3f} ms", flush=True)
for k in range(3):
    t0 = time.perf_counter(); est = h.estimate_nf(pg, cfg); t1 = time.perf_counter()
    print(f"estimate_nf {1e3*(t1-t0):.3f} ms", flush=True)
os.environ["HANF_NO_GRAPHS"] = "1"
for k in range(3):
    t0 = time.perf_counter(); est = h.estimate_nf(pg, cfg); t1 = time.perf_counter()
    print(f"estimate_nf (no graphs) {1e3*(t1-t0):.3f} ms", flush=True)
