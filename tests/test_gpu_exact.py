"""Exact neighbourhood function on the GPU (oracle.hpp:38-104 semantics)
against the oracle's all-pairs BFS, the reference's own exact_nf and the
clique-path closed form (oracle.hpp:107-113)."""
import numpy as np
import pytest

import paper_1011_5599_b200 as hanf

pytestmark = pytest.mark.gpu


def test_exact_matches_bfs_oracle(port):
    graphs = [hanf.gen_uniform_random(3000, 4, 9), hanf.gen_rmat(12, 8, 0.57, 0.19, 0.19, 2, 3),
              hanf.Graph.from_edges(5, [(0, 1), (1, 2), (2, 0), (3, 3)]),
              hanf.Graph.from_edges(1, []), hanf.gen_erdos_renyi(5000, 1.5, 4)]
    for g in graphs:
        want = port.exact_nf(g.num_nodes(), g.offsets(), g.arcs())
        got = hanf.exact_nf(g)
        assert [int(x) for x in want] == got.values, g.num_nodes()


def test_exact_matches_reference(ref):
    g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 5, 6)
    want = ref.exact_nf(ref.graph(g.num_nodes(), g.offsets(), g.arcs()))
    assert [int(x) for x in want] == hanf.exact_nf(g).values


def test_exact_clique_path_closed_form(port):
    for k, l in [(3, 5), (40, 7), (10, 300)]:
        g = hanf.gen_clique_path(k, l)
        got = hanf.exact_nf(g).values
        assert got == [port.clique_path_nf(k, l, t) for t in range(len(got))]
        assert len(got) - 1 == l + 1  # diameter of the clique-path graph


def test_exact_guard_and_empty():
    g = hanf.gen_uniform_random(2000, 3, 1)
    with pytest.raises(hanf.GuardError):
        hanf.exact_nf(g, max_nodes=1000)
    with pytest.raises(hanf.GuardError):
        hanf.exact_nf(g, max_work=1000)
    assert hanf.exact_nf(hanf.Graph(0)).values == [0]
