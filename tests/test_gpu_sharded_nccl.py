"""The production multi-GPU path (ShardedNfEngine over LocalCudaShard and
NCCL) on the one GPU a round has: world size 1, so the collectives are
trivial, but every piece runs for real - shard engines, device-buffer
views, stream hand-offs, the NCCL all-gathers and the changed-rows packets.
Equal to the single engine bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_engine_over_nccl_world1(hanf):
    import torch
    import torch.distributed as dist
    from paper_1011_5599_b200.sharded import ShardedNfEngine
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = hanf.gen_rmat(13, 16, 0.57, 0.19, 0.19, 3, 4)
        cfg = hanf.EngineConfig(bucket_bits=6, seed=17)
        single = hanf.estimate_nf(g, cfg)
        for delta_ratio in (16, 1):  # 1: changed-rows packets from step 2 on
            eng = ShardedNfEngine(g, cfg, 0, 1, delta_ratio=delta_ratio, delta_cap=g.num_nodes())
            est = eng.run_to_stabilisation()
            assert est.values == single.values and est.modified == single.modified
            if delta_ratio == 1:
                assert eng.delta_steps > 0
            with hanf.NfEngine(g, cfg) as e:
                e.run_to_stabilisation()
                assert np.array_equal(eng.local.engine.counters(), e.counters())
            eng.local.close()
    finally:
        dist.destroy_process_group()
