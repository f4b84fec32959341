"""Dev aid: bench.py's e2e leg in isolation; bisect what slows it in bench."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1011_5599_b200 as hanf
name, make, b = bench.workload(2)
g = make()
n, a = g.num_nodes(), g.num_arcs()
off_pin = torch.from_numpy(g.offsets().view("int64")).pin_memory()
arc_pin = torch.from_numpy(g.arcs().view("int32")).pin_memory()
pinned = hanf.Graph.__new__(hanf.Graph)
pinned._n = n
pinned._offsets = off_pin.numpy().view("uint64")
pinned._arcs = arc_pin.numpy().view("uint32")
cfg = hanf.EngineConfig(bucket_bits=b, seed=42)


def measure(tag):
    hanf.estimate_nf(pinned, cfg)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hanf.estimate_nf(pinned, cfg)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{tag:40s} " + " ".join(f"{t:.3f}" for t in ts), flush=True)


measure("fresh")
torch.cuda.set_device(0)
measure("+ set_device")
from paper_1011_5599_b200.sharded import ShardedNfEngine  # noqa: F401
measure("+ import sharded")
engine = hanf.NfEngine(g, hanf.EngineConfig(bucket_bits=b, seed=42, exact_sum=False))
measure("+ main engine alive")
stream = torch.cuda.ExternalStream(engine.stream(), device=torch.device("cuda", 0))
measure("+ external stream")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
measure("+ flush buffer")
for _ in range(5):
    engine.reset(); engine.step()
measure("+ steps")
with bench.ClockSampler(0) as clocks:
    for _ in range(5):
        engine.reset(); flush.zero_(); torch.cuda.synchronize(); engine.step()
measure("+ clock sampler")
engine.set_timing(True)
for _ in range(3):
    engine.reset(); flush.zero_(); torch.cuda.synchronize(); engine.step()
engine.timing(); engine.set_timing(False)
measure("+ timing pass")
engine.close()
measure("main engine closed")


def h2d(tag, t):
    d = torch.empty(t.numel(), dtype=t.dtype, device="cuda")
    for _ in range(3):
        d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{tag}: ptr % 2MiB = {t.data_ptr() % (2 << 20)}, {t.numel() * t.element_size() / dt / 1e9:.1f} GB/s", flush=True)


h2d("arc_pin (early)", arc_pin)
arc2 = torch.from_numpy(g.arcs().view("int32")).pin_memory()
h2d("arc_pin (late)", arc2)
big = [torch.empty(64 << 20, dtype=torch.uint8).pin_memory() for _ in range(3)]
arc3 = torch.from_numpy(g.arcs().view("int32")).pin_memory()
h2d("arc_pin (after other pinned blocks)", arc3)
pinned._arcs = arc3.numpy().view("uint32")
measure("estimate_nf with late pinned arcs")

