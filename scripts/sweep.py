"""Dev aid: union-kernel variant x L2 fetch granularity sweep on one config.
    python scripts/sweep.py CONFIG "v1,v2,..." "l2a,l2b,..." (or "ENV=VAL,..." instead of L2 fetch sizes)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1011_5599_b200 as h
cfgno = sys.argv[1]; variants = sys.argv[2].split(","); l2s = sys.argv[3].split(",")
if cfgno.startswith("rmat"):  # R-MAT scale k, config-2 parameters (dev sizes between 2 and 5)
    k = int(cfgno[4:])
    name, make, b = (f"R-MAT {k} (ef 16, ids permuted)",
                     lambda: h.gen_rmat(k, 16, 0.57, 0.19, 0.19, 1, 7), 6)
else:
    name, make, b = bench.workload(int(cfgno))
t0 = time.time(); g = make(); print(name, "gen", round(time.time() - t0, 1), "s", flush=True)
import ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for l2 in l2s:
    for v in variants:
        os.environ["HANF_GATHER"] = v
        if "=" in l2:
            k_, v_ = l2.split("=", 1); os.environ[k_] = v_
        else:
            os.environ["HANF_L2_FETCH"] = l2
        e = h.NfEngine(g, h.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
        e.reset(); e.step()
        e.set_timing(True)
        for _ in range(3):
            e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
        t = e.timing(); e.close()
        u = t["union_ms"] / t["steps"]
        fin = t["reduce_ms"] / t["steps"]
        print(f"config{cfgno} variant {v:>3} l2fetch {l2:>4}: union {u:.3f} ms  {g.num_arcs()/u/1e6:.1f} G arcs/s"
              f"  (+ finish {fin:.3f} ms)", flush=True)
