#!/usr/bin/env python
"""Generates tests/golden/*.json from the REFERENCE engine itself.

Run in the dev container, where /root/reference exists and oracle/_ref/
libhanf_ref.so is built from the reference's own headers (oracle/Makefile):

    make -C oracle && python tests/golden/make_golden.py

Every number in the fixtures comes from hyperanf::NfEngine / counter_* /
stats.hpp executing unmodified; the only code of ours involved is the
ctypes shim (oracle/ref_shim.cpp) and, for the synthetic R-MAT case, the
graph generator (pinned by the CSR hash stored beside it).  Floats are
stored with float.hex() so equality checks are bit-exact.

The recorded acceptance values at the end are quoted from the reference's
own recorded run, /root/reference/proj/test_output.txt (lines cited), and
re-derived here from the reference engine.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1011_5599_b200 as hanf  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_of(spec):
    kind = spec["kind"]
    if kind == "uniform_random":
        return hanf.gen_uniform_random(spec["n"], spec["d"], spec["seed"])
    if kind == "clique_path":
        return hanf.gen_clique_path(spec["k"], spec["l"])
    if kind == "edges":
        return hanf.Graph.from_edges(spec["n"], spec["edges"])
    if kind == "path":
        return hanf.Graph.from_edges(spec["n"], [(v, v + 1) for v in range(spec["n"] - 1)])
    if kind == "rmat":
        return hanf.gen_rmat(spec["scale"], spec["edge_factor"], 0.57, 0.19, 0.19, spec["seed"],
                             spec["permute_seed"])
    raise ValueError(kind)


CASES = [
    # test_engine.cpp:86-107 (balls), r in {5, 6}
    dict(name="balls60_r5", graph=dict(kind="uniform_random", n=60, d=3, seed=21),
         cfg=dict(bucket_bits=6, register_bits=5, seed=77), full_counters=True),
    dict(name="balls60_r6", graph=dict(kind="uniform_random", n=60, d=3, seed=21),
         cfg=dict(bucket_bits=6, register_bits=6, seed=77), full_counters=True),
    # test_engine.cpp:63-83 single arc, :109-133 3-path
    dict(name="single_arc", graph=dict(kind="edges", n=2, edges=[[0, 1]]),
         cfg=dict(bucket_bits=7, seed=9), full_counters=True),
    dict(name="path3", graph=dict(kind="edges", n=3, edges=[[0, 1], [1, 2]]),
         cfg=dict(bucket_bits=7, seed=5), full_counters=True),
    # test_engine.cpp:145-160 schedule independence graph
    dict(name="ur500", graph=dict(kind="uniform_random", n=500, d=5, seed=31),
         cfg=dict(bucket_bits=7, seed=8)),
    # test_engine.cpp:162-184 skipping / systolic
    dict(name="cp12_6", graph=dict(kind="clique_path", k=12, l=6), cfg=dict(bucket_bits=6, seed=4)),
    # test_engine.cpp:186-205 systolic activation on a 64-path
    dict(name="path64", graph=dict(kind="path", n=64), cfg=dict(bucket_bits=6, seed=2)),
    # test_engine.cpp:207-212
    dict(name="ur300_b5", graph=dict(kind="uniform_random", n=300, d=8, seed=3),
         cfg=dict(bucket_bits=5, seed=7)),
    # test_engine.cpp:135-143
    dict(name="ur400_s99", graph=dict(kind="uniform_random", n=400, d=6, seed=13),
         cfg=dict(bucket_bits=6, seed=99)),
    # acceptance.cpp:252-263 (test_output.txt:14): T = 11, final jump 71722.3
    dict(name="cp260_10_b8", graph=dict(kind="clique_path", k=260, l=10),
         cfg=dict(bucket_bits=8, seed=42)),
    # acceptance.cpp:174-197 (C3)
    dict(name="ur10000_b7", graph=dict(kind="uniform_random", n=10000, d=8, seed=777),
         cfg=dict(bucket_bits=7, seed=42)),
    # nodes of out-degree 1099 > 1024: exercises split (hub) nodes
    dict(name="cp1100_3_b6", graph=dict(kind="clique_path", k=1100, l=3),
         cfg=dict(bucket_bits=6, seed=42)),
    # every register width / bucket count the union kernels specialise
    *[dict(name=f"ur2000_b{b}_r{r}", graph=dict(kind="uniform_random", n=2000, d=5, seed=3),
           cfg=dict(bucket_bits=b, register_bits=r, seed=42))
      for b, r in [(4, 5), (5, 5), (6, 5), (7, 5), (8, 5), (10, 5), (4, 6), (5, 6), (7, 6),
                   (4, 7), (5, 7), (6, 7), (7, 7), (4, 8), (6, 8)]],
    # synthetic R-MAT (BASELINE config 2 generator at scale 14), pinned by CSR hash
    dict(name="rmat14", graph=dict(kind="rmat", scale=14, edge_factor=16, seed=1, permute_seed=7),
         cfg=dict(bucket_bits=6, seed=42)),
]


def trace_case(ref, case):
    g = csr_of(case["graph"])
    rg = ref.graph(g.num_nodes(), g.offsets(), g.arcs())
    cfg = case["cfg"]
    eng = ref.engine(rg, **cfg)
    rec = {"name": case["name"], "graph": case["graph"], "cfg": cfg,
           "n": g.num_nodes(), "arcs": g.num_arcs(),
           "csr_sha256": sha(np.concatenate([g.offsets().view(np.uint8), g.arcs().view(np.uint8)])),
           "sum0": float.hex(eng.sum_estimates()), "counters0_sha256": sha(eng.counters()),
           "steps": []}
    if case.get("full_counters"):
        rec["counters0"] = [int(x) for x in eng.counters()]
    for t in range(1, g.num_nodes() + 2):
        s, m = eng.step()
        c = eng.counters()
        step = {"t": t, "sum": float.hex(s), "modified": m, "counters_sha256": sha(c),
                "systolic": eng.systolic_active()}
        if case.get("full_counters"):
            step["counters"] = [int(x) for x in c]
        rec["steps"].append(step)
        if m == 0:
            break
    eng2 = ref.engine(rg, **cfg)
    vals, mods, _ = eng2.run()
    rec["run_values"] = [float.hex(v) for v in vals]
    rec["run_modified"] = mods
    if vals and vals[-1] > 0:
        mean, var, spid = ref.distance_distribution(vals)
        rec["stats"] = {"mean": float.hex(mean), "variance": float.hex(var),
                        "spid": float.hex(spid),
                        "ed": float.hex(ref.effective_diameter(vals, 0.9, False)),
                        "ied": float.hex(ref.effective_diameter(vals, 0.9, True))}
    return rec


def primitives(ref):
    """Estimates and unions of random counters (hll.hpp:122-180)."""
    rng = np.random.default_rng(20261019)
    out = []
    for b, r in [(4, 5), (6, 5), (7, 5), (8, 5), (10, 5), (6, 6), (7, 7), (6, 8)]:
        p_words = (1 << b) * r // 64 + (1 if ((1 << b) * r) % 64 else 0)
        m = 1 << b
        cases = []
        for rep in range(40):
            x = np.zeros(p_words, dtype=np.uint64)
            y = np.zeros(p_words, dtype=np.uint64)
            # geometric-ish register values, clamped to the register range
            for arr in (x, y):
                vals = np.minimum(rng.geometric(0.35 + 0.3 * (rep % 3) / 2, size=m) - 1,
                                  (1 << r) - 1)
                vals[rng.random(m) < (rep % 5) / 5.0] = 0
                for j, v in enumerate(vals):
                    ref.L.ref_write_register(oracle._u64p(arr), b, r, j, int(v))
            est = ref.counter_estimate(x, b, r)
            u = x.copy()
            changed = ref.L.ref_counter_union(oracle._u64p(u), oracle._u64p(y), b, r)
            cases.append({"x": [int(v) for v in x], "y": [int(v) for v in y],
                          "estimate_x": float.hex(est), "union": [int(v) for v in u],
                          "changed": bool(changed)})
        out.append({"b": b, "r": r, "cases": cases})
    return out


def main():
    ref = oracle.ref()
    ref.L.ref_write_register.argtypes = [oracle.POINTER(oracle.c_uint64), oracle.ctypes.c_uint,
                                         oracle.ctypes.c_uint, oracle.ctypes.c_uint,
                                         oracle.ctypes.c_uint]
    traces = [trace_case(ref, c) for c in CASES]
    with open(os.path.join(OUT, "engine_traces.json"), "w") as f:
        json.dump({"source": "reference NfEngine via oracle/_ref (make_golden.py)",
                   "cases": traces}, f, separators=(",", ":"))
    with open(os.path.join(OUT, "primitives.json"), "w") as f:
        json.dump({"source": "reference counter_estimate/counter_union via oracle/_ref",
                   "layouts": primitives(ref)}, f, separators=(",", ":"))
    # recorded acceptance values (the reference's own recorded run)
    recorded = {
        "source": "/root/reference/proj/test_output.txt",
        "unbiasedness_m64_worst": {"value": "0.01486", "line": 11,
                                   "graph": "gen_uniform_random(1000, 8, 4242)",
                                   "runs": "b=6, seeds 100..199"},
        "unbiasedness_m1024_worst": {"value": "0.004603", "line": 12,
                                     "runs": "b=10, seeds 100..199"},
        "concentration_m256": {"within2": 97, "within3": 100, "line": 13,
                               "runs": "b=8, seeds 300..399"},
        "clique_path_260_10": {"T": 11, "final_jump": "71722.3", "line": 14,
                               "cfg": "b=8, seed 42"},
        "spid": {"exact": ["5.03", "0.106"], "line": 23,
                 "reps": [["5.03", "0.026", "0.107", "0.044"],
                          ["5.02", "0.031", "0.107", "0.046"],
                          ["5.01", "0.032", "0.107", "0.046"]],
                 "graphs": ["gen_clique_path(252, 10)", "gen_uniform_random(1000, 20, 2020)"],
                 "runs": "b=7, seeds base+i, base = 500 + rep*1000, i < 100"},
        "estimate_all_ones_m16": {"value": "21.536", "source": "test_hll.cpp:86-94"},
    }
    with open(os.path.join(OUT, "recorded.json"), "w") as f:
        json.dump(recorded, f, indent=1)
    print("wrote", len(traces), "traces")


if __name__ == "__main__":
    main()
