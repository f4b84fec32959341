#!/usr/bin/env python
"""Benchmark of the B200 HyperANF iteration (BASELINE.json metric: arcs/s per
HyperANF iteration, and % of HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A "step" is one dense HyperANF iteration (iteration 1 from the seeded state:
every arc scanned, every counter read and written, estimates and N(1)
reduced) over the synthetic graph of BASELINE config C (default 2: R-MAT
scale 20).  The state is re-seeded and L2 flushed (256 MiB write) before
each timed step, outside the timed region; each step is timed with CUDA
events on the engine's stream.  One JSON line on rank 0.

  value     arcs/s, graph resident in HBM (device-timed dense iterations)
  e2e       arcs/s per iteration of a whole estimate_nf() through the C-ABI
            from pinned host CSR to N(t) on the host: upload, seeding, every
            iteration to stabilisation, read-back (wall clock)
  roofline  union sweep: SURVEY 8(d) algorithmic bytes per launch / the
            sweep's CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the reference engine (oracle/_ref) on this host's cores, on
            dense iterations of the same graph

--impl reference times the reference's own CPU engine (oracle/_ref, built
from /root/reference's headers) on e2e's metric: whole estimate_nf() runs,
all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HLL_SEED = 42
METRIC = "arcs/s per HyperANF iteration"


def workload(config: int):
    import paper_1011_5599_b200 as hanf
    if config == 1:
        return ("config1: directed G(n,p) n=65536, mean out-degree 8, no self-loops, seed 1; "
                "log2m=6", lambda: hanf.gen_erdos_renyi(65536, 8.0, 1), 6)
    if config == 2:
        return ("config2: R-MAT scale 20, edge factor 16, a=.57 b=.19 c=.19, self-loops/dups "
                "removed, ids permuted (seed 7); log2m=6",
                lambda: hanf.gen_rmat(20, 16, 0.57, 0.19, 0.19, 1, 7), 6)
    if config == 3:
        return ("config3: copying model n=2^24, power-law out-degree (2.1, mean 20, max 5000), "
                "copy prob 0.6, window +-2^12; log2m=7",
                lambda: hanf.gen_copying(1 << 24, 2.1, 20.0, 5000, 0.6, 1 << 12, 3), 7)
    if config == 4:
        return ("config4: Barabasi-Albert n=2^25, m=10, symmetric, ids permuted (seed 11); "
                "log2m=5", lambda: hanf.gen_barabasi_albert(1 << 25, 10, 4, 11), 5)
    if config == 5:
        return ("config5: R-MAT scale 28, edge factor 16, a=.57 b=.19 c=.19, ids permuted; "
                "log2m=6", lambda: hanf.gen_rmat(28, 16, 0.57, 0.19, 0.19, 1, 7), 6)
    raise SystemExit(f"unknown config {config}")


def algorithmic_bytes(n: int, a: int, words: int) -> int:
    """successor ids + gathered successor counters + offsets +
    own-counter read + next-counter write, per dense iteration."""
    return 4 * a + 8 * words * a + 8 * (n + 1) + 16 * words * n


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed
    region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                self.reasons |= self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            self._stop.wait(0.002)  # the timed loop is only tens of ms long

    def __enter__(self):
        if self._nv:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self._nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def ncu_traffic(config: int):
    """dram bytes per union-kernel launch from the committed ncu --set full
    summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "union_kernel_ncu.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"config{config}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference arm / cpu baseline (oracle/_ref: the reference engine itself)
# ---------------------------------------------------------------------------
def reference_arm(args, g, workload_name, b):
    import oracle
    ref = oracle.ref()
    threads = os.cpu_count() or 1
    rg = ref.graph(g.num_nodes(), g.offsets(), g.arcs())
    a = g.num_arcs()
    times, iters = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()  # estimate_nf = ctor (seeding) + run
        eng = ref.engine(rg, bucket_bits=b, seed=HLL_SEED, threads=threads)
        vals, mods, wall = eng.run()
        dt = time.perf_counter() - t0
        del eng
        if i >= args.warmup:
            times.append(dt)
            iters.append(len(vals))  # T recorded + the stabilising iteration
    value = a * sum(iters) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "arcs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": workload_name, "n": g.num_nodes(), "arcs": a, "log2m": b,
                   "hll_seed": HLL_SEED, "step": "one whole estimate_nf() run to "
                   "stabilisation (engine.hpp:233-275), arcs x iterations / wall time"},
        "cpu_baseline": {"value": value, "unit": "arcs/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"{args.steps} estimate_nf runs of {workload_name}, "
                                   f"threads={threads}, oracle/_ref (reference headers)"},
        "e2e": {"value": value, "unit": "arcs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(g, b, budget_s=12.0):
    """Reference engine, dense iteration 1 (same unit of work as `value`)."""
    import oracle
    if not oracle.have_ref():
        return None
    ref = oracle.ref()
    threads = os.cpu_count() or 1
    rg = ref.graph(g.num_nodes(), g.offsets(), g.arcs())
    steps, total = 0, 0.0
    start = time.perf_counter()
    while steps < 1 or (time.perf_counter() - start < budget_s and steps < 20):
        eng = ref.engine(rg, bucket_bits=b, seed=HLL_SEED, threads=threads)
        secs, _, _ = eng.timed_step()
        del eng
        total += secs
        steps += 1
    return {"value": g.num_arcs() * steps / total, "unit": "arcs/s", "cores": threads,
            "kind": "reference",
            "sample": f"{steps} dense iterations (iteration 1 from the seeded state) of the "
                      f"same graph, NfEngine::step() timed with steady_clock, threads={threads}"}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["peer", "collective"],
                    help="N>1: peer-push rows over NVLink from the union kernels "
                         "(hanf_shard_attach) or NCCL all-gathers")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    name, make_graph, b = workload(args.config)

    if args.impl == "reference":
        if rank != 0:
            return
        g = make_graph()
        reference_arm(args, g, name, b)
        return

    import torch
    import paper_1011_5599_b200 as hanf
    from paper_1011_5599_b200.sharded import ShardedNfEngine

    # BENCH_DIST_BACKEND=gloo runs the N>1 path with several ranks per GPU
    # (a functional check on a one-GPU box; NCCL needs distinct GPUs)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local_rank = local_rank % max(1, torch.cuda.device_count()) if backend != "nccl" else local_rank
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    g = make_graph()
    n, a = g.num_nodes(), g.num_arcs()
    cfg = hanf.EngineConfig(bucket_bits=b, seed=HLL_SEED, device=local_rank, exact_sum=False)
    if world > 1:
        sharded = ShardedNfEngine(g, cfg, rank, world, exchange=args.exchange)
        engine = sharded.local.engine
        do_step = sharded.step
    else:
        sharded = None
        engine = hanf.NfEngine(g, cfg)
        do_step = engine.step
    words = engine.params().words
    stream = torch.cuda.ExternalStream(engine.stream(), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    reset = sharded.reset if sharded is not None else engine.reset  # (shards: + barrier)
    for _ in range(args.warmup):
        reset()
        do_step()
    step_launches = 0
    total_ms = 0.0
    barrier()
    with ClockSampler(local_rank) as clocks:
        for _ in range(args.steps):
            reset()                              # untimed: back to the seeded state
            torch.cuda.synchronize(dev)
            launches_before = engine.launch_count()
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            if world == 1:
                # the L2 flush (untimed) keeps the GPU busy while the host
                # enqueues the step, so the events bracket the step's device
                # work only - no host launch latency inside the timed span
                flush.zero_()
                stream.wait_stream(torch.cuda.current_stream(dev))
                start.record(stream)
                engine.step_launch()
                end.record(stream)
                end.synchronize()
                rep = engine.step_complete()
            else:
                flush.zero_()                    # untimed: evict L2 (256 MiB > 126 MB)
                torch.cuda.synchronize(dev)
                start.record(stream)
                rep = do_step()
                end.record(stream)
                end.synchronize()
            total_ms += start.elapsed_time(end)
            step_launches += engine.launch_count() - launches_before  # the step's kernels only
    barrier()
    # kernel phases for the roofline: CUDA events between the kernels on the
    # engine stream (ungraphed steps, same kernels), same flush protocol
    engine.set_timing(True)
    for _ in range(max(3, min(args.steps, 10))):
        reset()
        flush.zero_()
        torch.cuda.synchronize(dev)
        do_step()
    timing = engine.timing()
    # the iterations after the dense ones, reported separately -
    # one whole run to stabilisation, device time of each step's sweep
    # (union / skip / worklist kernels) and of its finish, CUDA events
    run_profile = []
    if world == 1:
        engine.reset()
        engine.run_to_stabilisation()  # untimed: first launches of the tail kernels (lazy loading)
        engine.reset()
        prev = n
        while True:
            engine.set_timing(True)
            rep = do_step()
            t = engine.timing()
            kind = ("dense" if 2 * prev >= n else
                    "worklist or skip sweep (changed-successor probes)")
            run_profile.append({"t": len(run_profile) + 1, "modified": rep.modified, "kind": kind,
                                "sweep_ms": round(t["union_ms"], 4),
                                "finish_ms": round(t["reduce_ms"] + t["estimate_ms"], 4)})
            prev = rep.modified
            if rep.modified == 0 or len(run_profile) >= 4 * n + 8:
                break
    engine.set_timing(False)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = a * args.steps / (total_ms / 1e3)
    union_ms = timing["union_ms"] / max(1, timing["steps"])
    peak, peak_src = hbm_peak()
    if world > 1:
        # the rank's own sweep: its rows and their arcs (rank 0 reports; the
        # shards are arc-balanced by the id permutation / interleaving)
        lo, hi = sharded.ranges[rank]
        rank_arcs = (a // world if engine.device_buffers().relabelled  # rows interleaved by degree
                     else int(g.offsets()[hi]) - int(g.offsets()[lo]))
        B = algorithmic_bytes(hi - lo, rank_arcs, words)
    else:
        B = algorithmic_bytes(n, a, words)
    achieved = B / (union_ms / 1e3) / 1e9 if union_ms > 0 else None
    traffic = ncu_traffic(args.config) if world == 1 else None

    e2e = None
    if not args.no_e2e and world > 1:
        # whole sharded run through the public API: every rank page-locks
        # its copy of the CSR, creates its shard engine (uploads its rows),
        # attaches to the peers and iterates to stabilisation; wall time
        # max over ranks
        import torch.distributed as dist
        pinned = hanf.Graph(n, g.offsets().copy(), g.arcs().copy()).pin()
        e2e_cfg = hanf.EngineConfig(bucket_bits=b, seed=HLL_SEED, device=local_rank)
        runs, iters, wall = min(args.steps, 3), 0, 0.0
        for r in range(runs + 1):
            barrier()
            t0 = time.perf_counter()
            sh = ShardedNfEngine(pinned, e2e_cfg, rank, world, exchange=args.exchange)
            est = sh.run_to_stabilisation()
            dt = time.perf_counter() - t0
            sh.close()
            t = torch.tensor([dt], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if r > 0:  # run 0 warms the context and allocator
                wall += float(t.item())
                iters += est.iterations() + 1
        lo, hi = sharded.ranges[rank]
        blocks = (n + 63) // 64
        e2e = {"value": a * iters / wall, "unit": "arcs/s",
               "h2d_bytes_per_step": 8 * (n + 1) + 4 * (int(g.offsets()[hi]) - int(g.offsets()[lo])),
               "d2h_bytes_per_step": int(iters / runs * (16 + 8 * blocks)),
               "step": "whole sharded estimate_nf() per rank (upload of the rank's rows, "
                       "seed, every iteration, read-back), max over ranks; bytes per rank"}
    if not args.no_e2e and world == 1:
        # whole estimate_nf through the C-ABI from pinned host memory: the
        # caller's CSR (fresh numpy arrays) page-locked in place with
        # Graph.pin() (hanf_pin_host).  torch.pin_memory() buffers are not
        # used: on these VMs their H2D rate varies 21-55 GB/s from buffer to
        # buffer, registered huge-page memory holds 55 (profiles/r01_h2d.md)
        pinned = hanf.Graph(n, g.offsets().copy(), g.arcs().copy()).pin()
        e2e_cfg = hanf.EngineConfig(bucket_bits=b, seed=HLL_SEED, device=local_rank)
        hanf.estimate_nf(pinned, e2e_cfg)     # warm (context, allocator)
        runs, iters, wall = min(args.steps, 5), 0, 0.0
        for _ in range(runs):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            est = hanf.estimate_nf(pinned, e2e_cfg)
            wall += time.perf_counter() - t0
            if os.environ.get("BENCH_DEBUG"):
                print(f"e2e run {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr)
            iters += est.iterations() + 1       # + the stabilising iteration
        blocks = (n + 63) // 64
        per_run_iters = iters / runs
        e2e = {"value": a * iters / wall, "unit": "arcs/s",
               "h2d_bytes_per_step": 8 * (n + 1) + 4 * a,
               "d2h_bytes_per_step": int(per_run_iters * (16 + 8 * blocks)
                                         + 16 * (est.iterations() + 1)),
               "step": "whole estimate_nf() (upload, seed, %d iterations, read-back) per step"
                       % round(per_run_iters)}

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        try:
            cpu = cpu_baseline(g, b)
        except Exception as exc:  # the checker must not take the bench down
            cpu = {"value": None, "error": str(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "arcs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": name, "n": n, "arcs": a, "log2m": b, "register_bits": 5,
                       "words_per_counter": words, "hll_seed": HLL_SEED,
                       "parallelism": f"node-range shards x{world}" if world > 1 else "1 GPU",
                       "exchange": (sharded.exchange + (f" (fallback: {sharded.fallback})"
                                                        if sharded.fallback else ""))
                                   if sharded is not None else None,
                       "step": "dense iteration 1 (all arcs) incl. estimates, N(t) total, "
                               "D2H report; re-seed + L2 flush outside the timed region; "
                               "events bracket the step's device work (launch enqueued "
                               "during the flush)",
                       "l2": "flushed before every timed step (256 MiB write)",
                       "sum_mode": "device (deterministic tree)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": "union_kernel (successor gather + broadword max + fused estimator)",
                         "kernel_ms": union_ms, "algorithmic_bytes": B,
                         "peak_source": peak_src,
                         "phases_ms": {"union": timing["union_ms"] / max(1, timing["steps"]),
                                       "estimate": timing["estimate_ms"] / max(1, timing["steps"]),
                                       "finish": timing["reduce_ms"] / max(1, timing["steps"])}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "run_profile": run_profile or None,
            "gpu_launches": step_launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if sharded is not None:
        sharded.close()
    else:
        engine.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
