"""One engine over several devices (hanf_create_multi, EngineConfig.devices):
node-range shards driven from one host thread, exchanging rows by the
peer-push, with a device-side barrier (stream event waits) per step.  On
the one-GPU test box the shards share device 0 (no kernel waits on another:
the barrier is between kernels).  Every step is bit-identical to the
oracle (counters, modified, N(t)), as the reference requires of any
schedule (test_engine.cpp:145-184)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices,relabel", [((0, 0), None), ((0, 0, 0), None),
                                             ((0, 0, 0, 0), "1"), ((0,) * 8, "1"),
                                             ((0, 0, 0, 0), "0")])
def test_multi_device_lockstep(hanf, port, monkeypatch, devices, relabel):
    if relabel is not None:
        monkeypatch.setenv("HANF_RELABEL", relabel)
    g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 1, 7)
    cfg = hanf.EngineConfig(bucket_bits=6, seed=42, devices=devices)
    ref = port.engine(g.num_nodes(), g.offsets(), g.arcs(), bucket_bits=6, seed=42)
    with hanf.NfEngine(g, cfg) as eng:
        assert eng.sum_estimates() == ref.sum_estimates()
        for t in range(1, 200):
            rep = eng.step()
            s, m = ref.step()
            assert (rep.sum, rep.modified) == (s, m), f"t={t}"
            assert np.array_equal(eng.counters(), ref.counters()), f"t={t}"
            assert eng.iteration() == t
            if m == 0:
                break
        eng.reset()
        est = eng.run_to_stabilisation()
        want = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=42))
        assert est.values == want.values and est.modified == want.modified
        eng.reseed(7)
        est7 = eng.run_to_stabilisation()
        assert est7.values == hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=7)).values


def test_multi_device_launch_complete_and_snapshot(hanf, tmp_path):
    g = hanf.gen_uniform_random(5000, 6, 3)
    one = hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=7, seed=1))
    many = hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=7, seed=1, devices=(0, 0, 0)))
    for _ in range(3):
        many.step_launch()
        r = many.step_complete()
        assert r == one.step()
    one.save_counters(tmp_path / "a.hca")
    many.save_counters(tmp_path / "b.hca")
    assert (tmp_path / "a.hca").read_bytes() == (tmp_path / "b.hca").read_bytes()
    with pytest.raises(ValueError):
        many.restore_counters(tmp_path / "a.hca")
    one.close()
    many.close()


def test_multi_device_config2_full_size(hanf):
    """Config 2 (R-MAT scale 20) as 4 shards: the whole run equals the single
    engine's bit for bit."""
    g = hanf.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7, device=0)
    a = hanf.estimate_nf(g, hanf.EngineConfig(bucket_bits=6, seed=42))
    with hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=6, seed=42, devices=(0, 0, 0, 0))) as e:
        b = e.run_to_stabilisation()
    assert a.values == b.values and a.modified == b.modified
