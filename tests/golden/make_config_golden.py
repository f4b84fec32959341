#!/usr/bin/env python
"""At-size parity fixtures: the REFERENCE engine (oracle/_ref, compiled from
the reference's own headers) run to stabilisation on BASELINE configs 1, 3,
4 and 5 at their exact specifications, one JSON per config in tests/golden/.

    python tests/golden/make_config_golden.py [CONFIG ...]      (default 1 3 4 5)

Run on the B200 host (16 cores, 196 GB: config 5 needs ~65 GB and ~15 min;
this container has neither) and commit the JSON files it writes:

    gpurun -- 'python tests/golden/make_config_golden.py 5 > gpurun_out/g5.log'

Per recorded iteration t the fixture holds the reference's modified count,
N(t) as float.hex, and the digest of the whole counter array
(oracle.port().counter_digest: order-independent mix over (row, words)),
plus the clamped N(t) series of run_to_stabilisation (engine.hpp:233-275),
the effective diameter (alpha 0.9, both variants) and spid (stats.hpp).
The graph is recorded by its CSR digest, so the GPU tests can check they
iterate the same graph.  Graphs: config 5 from the oracle's R-MAT
restatement (oracle/hanf_oracle_gen.c, pinned to the package generators by
tests/test_oracle_gen.py); configs 1, 3, 4 from the package's host
generators (graph input only; their CSR digests are recorded).
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SPEC = {
    1: dict(b=6, graph="gen_erdos_renyi(65536, 8.0, 1)"),
    3: dict(b=7, graph="gen_copying(1 << 24, 2.1, 20.0, 5000, 0.6, 1 << 12, 3)"),
    4: dict(b=5, graph="gen_barabasi_albert(1 << 25, 10, 4, 11)"),
    5: dict(b=6, graph="oracle gen_rmat(28, 16, 0.57, 0.19, 0.19, 1, 7)"),
}


def digest_every(config, t):
    if config != 3:
        return True
    return t <= 12 or t % 64 == 0


def graph_for(config):
    P = oracle.port()
    if config == 5:
        return P.gen_rmat(28, 16, 0.57, 0.19, 0.19, 1, 7)
    import paper_1011_5599_b200 as hanf
    g = eval("hanf." + SPEC[config]["graph"])
    return g.num_nodes(), g.offsets(), g.arcs()


def run(config):
    t0 = time.time()
    P, R = oracle.port(), oracle.ref()
    n, off, succ = graph_for(config)
    a = int(off[-1])
    csr = P.csr_digest(n, off, succ)
    rg = R.graph_sorted(n, off, succ)
    del off, succ
    b = SPEC[config]["b"]
    threads = len(os.sched_getaffinity(0))
    eng = R.engine(rg, bucket_bits=b, seed=42, threads=threads)
    W = eng.words if hasattr(eng, "words") else None
    ptr, wc = eng.counters_ptr()
    W = wc // n
    print(f"config {config}: n={n} a={a} W={W} setup {time.time() - t0:.1f} s", flush=True)
    iters = [{"t": 0, "modified": n, "sum": eng.sum_estimates().hex(),
              "digest": P.counter_digest(ptr, n, W)}]
    while True:
        ts = time.time()
        s, m = eng.step()
        t = len(iters)
        rec = {"t": t, "modified": int(m), "sum": s.hex()}
        if digest_every(config, t) or m == 0:
            ptr, _ = eng.counters_ptr()
            rec["digest"] = P.counter_digest(ptr, n, W)
        iters.append(rec)
        if t <= 12 or t % 100 == 0 or m == 0:
            print(f"  t={t} modified={m} sum={s:.6e} ({time.time() - ts:.1f} s)", flush=True)
        if m == 0:
            break
        if t > n + 1:
            raise RuntimeError("iteration cap")
    # run_to_stabilisation's record: N(0..T) without the stabilising step,
    # clamped to the running max (engine.hpp:252-270)
    vals = [float.fromhex(r["sum"]) for r in iters[:-1]]
    for i in range(1, len(vals)):
        vals[i] = max(vals[i], vals[i - 1])
    mean, var, spid = R.distance_distribution(vals)
    out = {
        "config": config, "spec": SPEC[config], "n": n, "arcs": a, "words": W,
        "hll_seed": 42, "register_bits": 5, "csr_digest": csr,
        "iterations": iters,
        "values": [v.hex() for v in vals],
        "effective_diameter": R.effective_diameter(vals, 0.9, False),
        "effective_diameter_interpolated": R.effective_diameter(vals, 0.9, True).hex(),
        "spid": spid.hex(), "mean": mean.hex(), "variance": var.hex(),
        "source": "oracle/_ref (the reference engine from its own headers), threads=%d, "
                  "%.0f s" % (threads, time.time() - t0),
    }
    with open(os.path.join(OUT, f"config{config}_trace.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(f"config {config}: T={len(vals) - 1} done in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    for c in [int(x) for x in sys.argv[1:]] or [1, 3, 4, 5]:
        run(c)
