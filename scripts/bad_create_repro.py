import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as hanf
os.environ["HANF_PIPELINE"] = sys.argv[1]
g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 2, 3)
cfg = hanf.EngineConfig(bucket_bits=6, seed=21)
ref = hanf.estimate_nf(g, cfg)
def check(tag):
    with hanf.NfEngine(g, cfg) as e:
        v = e.run_to_stabilisation().values
    print(tag, v == ref.values, v[:2], flush=True)
check("fresh")
with hanf.NfEngine(g, cfg) as e:
    e.step(); e.reset()
    print("after reset", e.run_to_stabilisation().values == ref.values)
    e.reseed(22); e.run_to_stabilisation()
check("after reseed engine")
for i in range(4):
    check(f"again {i}")
arcs = g.arcs().copy()
arcs[len(arcs) // 2] = g.num_nodes() + 5
bad = hanf.Graph(g.num_nodes(), g.offsets().copy(), arcs)
try:
    hanf.NfEngine(bad, cfg)
except ValueError as exc:
    print("ValueError:", exc)
for i in range(4):
    check(f"after bad {i}")
