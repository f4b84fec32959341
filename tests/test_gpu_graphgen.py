"""GPU graph construction builds the host builders'
CSR bit for bit: Graph::from_edges semantics (rows sorted, duplicates
collapsed, self-loops kept) and the R-MAT generator of configs 2 and 5."""
import numpy as np
import pytest

import paper_1011_5599_b200 as hanf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale,ef,seed,pseed", [(4, 4, 1, 7), (12, 16, 3, 5), (16, 16, 1, 7),
                                                 (20, 16, 1, 7)])
def test_rmat_gpu_equals_host(scale, ef, seed, pseed):
    a = hanf.gen_rmat(scale, ef, 0.57, 0.19, 0.19, seed, pseed)
    b = hanf.gen_rmat(scale, ef, 0.57, 0.19, 0.19, seed, pseed, device=0)
    assert a.num_nodes() == b.num_nodes()
    assert np.array_equal(a.offsets(), b.offsets())
    assert np.array_equal(a.arcs(), b.arcs())


def test_from_edges_gpu_equals_host():
    rng = np.random.default_rng(5)
    for n, m in [(1, 0), (7, 40), (1000, 20000), (70000, 500000)]:
        e = rng.integers(0, n, size=(m, 2))
        if m:
            e[: m // 10, 1] = e[: m // 10, 0]          # self-loops (kept by from_edges)
            e[m // 10: m // 5] = e[: m // 10]          # duplicates (collapsed)
        a = hanf.Graph.from_edges(n, e)
        b = hanf.Graph.from_edges(n, e, device=0)
        assert np.array_equal(a.offsets(), b.offsets()) and np.array_equal(a.arcs(), b.arcs())


def test_from_edges_gpu_rejects_bad_endpoint():
    src = np.array([0, 5], dtype=np.uint32)
    dst = np.array([1, 2], dtype=np.uint32)
    import ctypes
    from ctypes import POINTER, c_uint32, c_void_p
    h = c_void_p()
    st = hanf._lib.lib().hanf_graph_from_edges_gpu(0, 3, src.ctypes.data_as(POINTER(c_uint32)),
                                                    dst.ctypes.data_as(POINTER(c_uint32)), 2,
                                                    ctypes.byref(h))
    assert st != 0 and not h.value
