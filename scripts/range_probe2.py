import os, sys
sys.path.insert(0, "/root/repo")
import torch, bench
import paper_1011_5599_b200 as h
g = bench.make_graph(5, device=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for layout in ("packed", "bytes"):
    os.environ["HANF_LAYOUT"] = layout
    e = h.NfEngine(g, h.EngineConfig(bucket_bits=6, seed=42, exact_sum=False))
    for spec in ["", "0,0", "0,2097152", "2097152,4294967295", "0,8388608", "8388608,4294967295"]:
        if spec: os.environ["HANF_DBG_RANGE"] = spec
        else: os.environ.pop("HANF_DBG_RANGE", None)
        e.reset(); e.step()
        e.set_timing(True)
        for _ in range(3):
            e.reset(); flush.zero_(); torch.cuda.synchronize(); e.step()
        t = e.timing(); e.set_timing(False)
        print(layout, spec or "all", round(t["union_ms"] / t["steps"], 2), flush=True)
    e.close()
