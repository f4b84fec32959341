import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_5599_b200 as hanf
os.environ["HANF_PIPELINE"] = sys.argv[1]
variant = sys.argv[2]
g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 2, 3)
cfg = hanf.EngineConfig(bucket_bits=6, seed=21)
ref = hanf.estimate_nf(g, cfg)
def check(tag):
    with hanf.NfEngine(g, cfg) as e:
        v = e.run_to_stabilisation().values
    print(sys.argv[1], variant, tag, v == ref.values, v[:2], flush=True)
with hanf.NfEngine(g, cfg) as e:
    if variant == "reseed":
        e.reseed(22); e.run_to_stabilisation()
    elif variant == "runs":
        for _ in range(4):
            e.reset(); e.run_to_stabilisation()
    elif variant == "other":
        pass
if variant == "other":
    hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=22))
check("next")
check("next2")
