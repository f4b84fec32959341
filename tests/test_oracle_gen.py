"""Pins of the bench/reference-arm checkers (oracle/hanf_oracle_gen.c and
the ref_shim sample): the oracle's R-MAT restatement builds the same CSR as
the package's host and device generators; the reference Graph built from a
sorted CSR equals Graph::from_edges'; the bounded step sample is exactly
NfEngine::step's per-node body (engine.hpp:157-184)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle


def _same_csr(g, n, off, succ):
    return g.num_nodes() == n and np.array_equal(g.offsets(), off) and \
        np.array_equal(g.arcs(), succ)


@pytest.mark.parametrize("scale,ef,seed,pseed", [(12, 16, 1, 7), (14, 8, 3, 5), (17, 16, 1, 7)])
def test_oracle_rmat_equals_host_generator(hanf, port, scale, ef, seed, pseed):
    n, off, succ = port.gen_rmat(scale, ef, 0.57, 0.19, 0.19, seed, pseed, threads=3)
    g = hanf.gen_rmat(scale, ef, 0.57, 0.19, 0.19, seed, pseed)
    assert _same_csr(g, n, off, succ)
    # thread count never changes the graph
    n2, off2, succ2 = port.gen_rmat(scale, ef, 0.57, 0.19, 0.19, seed, pseed, threads=1)
    assert np.array_equal(off, off2) and np.array_equal(succ, succ2)


def test_oracle_rmat_config2_digest(hanf, port):
    """Config 2 exactly (scale 20, seed 1, permutation seed 7): the digest of
    the oracle's CSR equals the package host generator's."""
    n, off, succ = port.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7)
    assert off[-1] == 16086049
    g = hanf.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7)
    assert port.csr_digest(n, off, succ) == port.csr_digest(n, g.offsets(), g.arcs())


def test_counter_digest_is_order_and_thread_independent(port):
    rng = np.random.default_rng(3)
    w = rng.integers(0, 2**63, size=5 * 1000, dtype=np.uint64)
    d1 = port.counter_digest(w, 1000, 5, threads=1)
    assert d1 == port.counter_digest(w, 1000, 5, threads=7)
    w2 = w.copy()
    w2[17] ^= np.uint64(1)
    assert port.counter_digest(w2, 1000, 5) != d1


ref_only = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


@ref_only
def test_ref_graph_from_sorted_csr_equals_from_edges(hanf):
    R = oracle.ref()
    g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 1, 7)
    a = R.graph_sorted(g.num_nodes(), g.offsets(), g.arcs())
    b = R.graph(g.num_nodes(), g.offsets(), g.arcs())
    oa, sa = a.csr()
    ob, sb = b.csr()
    assert np.array_equal(oa, ob) and np.array_equal(sa, sb)
    bad = g.arcs().copy()
    bad[0], bad[1] = bad[1], bad[0]  # row 0 unsorted (if it has two arcs)
    if g.offsets()[1] >= 2 and bad[0] != bad[1]:
        with pytest.raises(ValueError):
            R.graph_sorted(g.num_nodes(), g.offsets(), bad)


@ref_only
def test_ref_step_sample_is_the_step_body(hanf):
    """Samples over a partition of [0, n) leave next_ equal to the counters
    of a real NfEngine::step, with the same changed count and block sums."""
    R = oracle.ref()
    g = hanf.gen_rmat(14, 16, 0.57, 0.19, 0.19, 1, 7)
    n = g.num_nodes()
    rg = R.graph_sorted(n, g.offsets(), g.arcs())
    full = R.engine(rg, bucket_bits=6, seed=42, threads=2)
    total, modified = full.step()
    sampled = R.engine(rg, bucket_bits=6, seed=42, threads=2)
    cuts = [0, 64 * 37, 64 * 100, 9000, n]  # block-aligned and not
    arcs = changed = 0
    for lo, hi in zip(cuts, cuts[1:]):
        _, a, _, ch = sampled.step_sample(lo, hi, 3)
        arcs += a
        changed += ch
    assert arcs == g.num_arcs() and changed == modified
    assert np.array_equal(sampled.next_counters(), full.counters())
    # one full-range sample: the same block sums summed in the same order
    one = R.engine(rg, bucket_bits=6, seed=42, threads=2)
    _, _, s, _ = one.step_sample(0, n, 4)
    assert s == total
