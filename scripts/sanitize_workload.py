"""Workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the engine paths on small graphs, each checked against the
oracle so a run also proves the results.
    compute-sanitizer --tool T python scripts/sanitize_workload.py PATH
PATH: dense | packed | worklist | summary | segments | peer | multi | relabel | hubs"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1011_5599_b200 as h

path = sys.argv[1]
env = {"packed": {"HANF_LAYOUT": "packed"}, "worklist": {"HANF_SPARSE": "1"}, "summary": {"HANF_SUMMARY": "1"},
       "segments": {"HANF_SEGMENTS": "1"}, "relabel": {"HANF_RELABEL": "1"},
       "multi": {}, "peer": {"HANF_RELABEL": "1"}}.get(path, {})
os.environ.update(env)
os.environ.setdefault("HANF_NO_GRAPHS", "1")  # plain launches: the tools see every kernel
g = (h.gen_clique_path(1500, 4) if path == "hubs"
     else h.gen_rmat(12, 16, 0.57, 0.19, 0.19, 1, 7))
cfg = h.EngineConfig(bucket_bits=6, seed=42,
                     devices=(0, 0) if path == "multi" else ((0,) * 4 if path == "peer" else ()))
port = oracle.port()
ref = port.engine(g.num_nodes(), g.offsets(), g.arcs(), bucket_bits=6, seed=42)
with h.NfEngine(g, cfg) as e:
    for t in range(1, 500):
        r = e.step()
        s, m = ref.step()
        assert (r.sum, r.modified) == (s, m), (t, r, s, m)
        assert np.array_equal(e.counters(), ref.counters()), t
        if m == 0:
            break
print(f"{path}: {t} steps bit-exact, {e.launch_count() if False else ''}ok")
