import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from ctypes import c_uint64, c_void_p, c_double, POINTER
import numpy as np
import paper_1011_5599_b200 as h
L = h._lib.lib()
for (g, b) in [(h.gen_uniform_random(1500, 3, 4), 8), (h.gen_uniform_random(1500, 3, 4), 6)]:
    for seed in (1000, 1001):
        e = h.NfEngine(g, h.EngineConfig(bucket_bits=b, seed=seed))
        ms = []
        for _ in range(12):
            r = e.step(); ms.append(r.modified)
            if r.modified == 0: break
        print("single", b, seed, ms)
    view, cfg = g.view(), h.EngineConfig(bucket_bits=b, seed=1000, max_iterations=12).to_c()
    seeds = (c_uint64 * 2)(1000, 1001)
    hh = c_void_p()
    h._lib.check(L.hanf_create_batch(ctypes.byref(view), ctypes.byref(cfg), seeds, 2, ctypes.byref(hh)))
    cap = 64
    vals = np.empty(2 * cap); mods = np.empty(2 * cap, dtype=np.uint64); lens = (c_uint64 * 2)()
    st = L.hanf_run_batch(hh, vals.ctypes.data_as(POINTER(c_double)), mods.ctypes.data_as(POINTER(c_uint64)), cap, lens)
    print("batch st", st, L.hanf_last_error(), list(lens), [list(mods[k*cap:k*cap+min(lens[k],14)]) for k in range(2)])
    L.hanf_destroy(hh)
