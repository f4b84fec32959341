"""The synthetic R-MAT generator (BASELINE configs 2 and 5) against an
independent numpy restatement of its stream: draw i descends `scale`
levels with 16 bits of hash3(seed, i, level/4) per level; ids go through
a 4-round Feistel bijection; self-loops and duplicate arcs are dropped and
rows sorted (graph.hpp:29-44 semantics).  The GPU builder must produce the
same CSR (tests/test_gpu_graphgen.py)."""
import numpy as np

import paper_1011_5599_b200 as hanf

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(33))
        z = z * np.uint64(0xFF51AFD7ED558CCD)
        z = z ^ (z >> np.uint64(33))
        z = z * np.uint64(0xC4CEB9FE1A85EC53)
        z = z ^ (z >> np.uint64(33))
    return z


def hash3(seed, key, k):
    with np.errstate(over="ignore"):
        a = mix64(np.uint64(seed) ^ np.uint64(0x5851F42D4C957F2D))
        b = mix64(np.asarray(key, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(k))
    return mix64(a ^ b)


def feistel(x, bits, seed):
    lbits, rbits = bits // 2, bits - bits // 2
    with np.errstate(over="ignore"):
        keys = [mix64(np.uint64(seed * 4 + i + 0x7F4A7C15)) for i in range(4)]
    x = np.asarray(x, dtype=np.uint64)
    l, r = x >> np.uint64(rbits), x & np.uint64((1 << rbits) - 1)
    lb, rb = lbits, rbits
    for i in range(4):
        f = mix64(r ^ keys[i]) & np.uint64((1 << lb) - 1)
        l, r = r, l ^ f
        lb, rb = rb, lb
    return (l << np.uint64(rb)) | r


def rmat_numpy(scale, ef, a, b, c, seed, pseed):
    n = 1 << scale
    i = np.arange(n * ef, dtype=np.uint64)
    ta, tb, tc = int(a * 65536.0), int((a + b) * 65536.0), int((a + b + c) * 65536.0)
    u = np.zeros_like(i)
    v = np.zeros_like(i)
    h = None
    for level in range(scale):
        if level % 4 == 0:
            h = hash3(seed, i, level // 4)
        r = (h >> np.uint64(16 * (level % 4))) & np.uint64(0xFFFF)
        bu = r >= tb
        bv = ((r >= ta) & (r < tb)) | (r >= tc)
        u = (u << np.uint64(1)) | bu.astype(np.uint64)
        v = (v << np.uint64(1)) | bv.astype(np.uint64)
    su, sv = feistel(u, scale, pseed), feistel(v, scale, pseed)
    keep = su != sv
    keys = np.unique((su[keep] << np.uint64(32)) | sv[keep])
    src = (keys >> np.uint64(32)).astype(np.int64)
    off = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(off, src + 1, 1)
    return np.cumsum(off, dtype=np.uint64), (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def test_rmat_stream_matches_restatement():
    for scale, ef, seed, pseed in [(8, 8, 1, 7), (11, 16, 3, 5), (12, 4, 9, 2)]:
        off, arcs = rmat_numpy(scale, ef, 0.57, 0.19, 0.19, seed, pseed)
        g = hanf.gen_rmat(scale, ef, 0.57, 0.19, 0.19, seed, pseed)
        assert np.array_equal(g.offsets(), off)
        assert np.array_equal(g.arcs(), arcs)
