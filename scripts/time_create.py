"""Dev aid: where does estimate_nf's wall time go (config 2, pinned CSR)?"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1011_5599_b200 as h
g = h.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7)
off = torch.from_numpy(g.offsets().view("int64")).pin_memory()
arc = torch.from_numpy(g.arcs().view("int32")).pin_memory()
pg = h.Graph(g.num_nodes(), off.numpy().view("uint64"), arc.numpy().view("uint32"))
torch.cuda.init()
for ex in (True, False):
    cfg = h.EngineConfig(bucket_bits=6, seed=42, exact_sum=ex)
    for k in range(3):
        t0 = time.perf_counter(); e = h.NfEngine(pg, cfg); t1 = time.perf_counter()
        est = e.run_to_stabilisation(); t2 = time.perf_counter(); e.close(); t3 = time.perf_counter()
        print(f"exact={ex} create {1e3*(t1-t0):.2f} ms  run {1e3*(t2-t1):.2f} ms ({est.iterations()} it)  destroy {1e3*(t3-t2):.2f} ms")
    e = h.NfEngine(pg, cfg)
    for t in range(9):
        t0 = time.perf_counter(); r = e.step(); t1 = time.perf_counter()
        print(f"  step {t+1}: {1e3*(t1-t0):.3f} ms modified {r.modified}")
        if r.modified == 0: break
    e.close()
print("--- second engine, ungraphed")
os.environ["HANF_NO_GRAPHS"] = "1"
for rep in range(2):
    e = h.NfEngine(pg, h.EngineConfig(bucket_bits=6, seed=42, exact_sum=False))
    for t in range(9):
        t0 = time.perf_counter(); r = e.step(); t1 = time.perf_counter()
        print(f"  step {t+1}: {1e3*(t1-t0):.3f} ms modified {r.modified}")
        if r.modified == 0: break
    e.close()
