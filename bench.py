#!/usr/bin/env python3
"""bench.py — MEMQSim hot path on B200: gates/s and circuit time at n qubits.

Default workload (BASELINE.json configs[1]): 30-qubit QFT (2220 gates) from
|0...0>, compressed-chunk store fully resident in HBM, c=16, eb=1e-5.
A step = one circuit execution through the staged pipeline: store init
(store.cpp:26-81) + every stage's decode → fused gate passes → encode
(pipeline.cpp:128-314), ending with the final compressed store in HBM.

  python bench.py [--gpus N --steps K --warmup W]          engine arm
  python bench.py --impl reference [...]                   reference CPU arm

Multi-GPU (torchrun, one rank per GPU): in this round every rank runs its
own replica of the workload ("replicas only" until the sharded
exchange lands), value = all ranks' gates / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "gates/sec and circuit time at n qubits (1/2/4/8 B200); comp. ratio; fidelity"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--circuit", default="qft")
    ap.add_argument("--n", type=int, default=30)
    ap.add_argument("--c", type=int, default=16)
    ap.add_argument("--m", type=int, default=30)
    ap.add_argument("--eb", type=float, default=1e-5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fidelity", action="store_true",
                    help="skip the uncompressed fp64 reference run used for the fidelity figure")
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="seconds of reference CPU work per sample")
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--strict-passes", action="store_true",
                    help="every gate qubit inside the pass tile (no relaxed diagonal units)")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: shard ONE circuit over the ranks by global qubits with NCCL "
                         "exchange of compressed chunks (strong scaling) instead of replicas")
    ap.add_argument("--residency", default="hbm", choices=["hbm", "host"],
                    help="compressed store in HBM (config 2) or pinned host memory (config 3)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.t0 = self.t1 = None

    def mark_begin(self):
        import datetime
        self.t0 = datetime.datetime.now()

    def mark_end(self):
        import datetime
        self.t1 = datetime.datetime.now()

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        import datetime
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f")
            except ValueError:
                ts = None
            # samples inside the timed region only (plus one sampling period)
            if ts and self.t0 and self.t1 and not (
                    self.t0 - datetime.timedelta(milliseconds=100) <= ts
                    <= self.t1 + datetime.timedelta(milliseconds=100)):
                continue
            f = f[1:]
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------- reference --
def reference_sample(circuit, n, c, m, eb, budget_s, workers=0):
    """Time the UNMODIFIED reference qzsim::run (oracle/_ref/libqzref.so) on a
    bounded sample of the same workload.  At n=30 one reference stage sweep
    alone takes ~40 s on 16 cores, so the sample is the same circuit family
    run in full at the largest n_s <= n whose run fits budget_s, with the
    same c, m (capped at n_s) and eb; gates/s is then scaled by 2^(n_s - n)
    (every gate and codec sweep touches 2^n amplitudes).  The time is the
    reference's own report.wall_seconds (pipeline.cpp:158-290)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracles import Reference  # baseline infrastructure only
    from paper_2309_16979_b200 import circuits
    ref = Reference()
    ns = max(c + 2, min(n, 20))
    last = None
    while True:
        gates = circuits.make(circuit, ns)
        t = time.time()
        r = ref.run(ns, gates, c, min(m, ns), eb, workers=workers, depth=2, strategy=2)
        el = time.time() - t
        last = {"n_sample": ns, "gates": len(gates), "wall_seconds": r["wall_seconds"],
                "elapsed": el, "gates_per_s_sample": len(gates) / r["wall_seconds"],
                "gates_per_s": len(gates) / r["wall_seconds"] * 2.0 ** (ns - n),
                "digest": r["digest"], "stages": r["stages"]}
        if ns >= n or el * 4.5 > budget_s:
            return last
        ns += 2


def reference_sample_fixed(args, first):
    """Repeat the sample at the n_s chosen by the first step."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracles import Reference
    from paper_2309_16979_b200 import circuits
    ns = first["n_sample"]
    gates = circuits.make(args.circuit, ns)
    t = time.time()
    r = Reference().run(ns, gates, args.c, min(args.m, ns), args.eb, workers=0, depth=2, strategy=2)
    return {"n_sample": ns, "gates": len(gates), "wall_seconds": r["wall_seconds"],
            "elapsed": time.time() - t, "gates_per_s_sample": len(gates) / r["wall_seconds"],
            "gates_per_s": len(gates) / r["wall_seconds"] * 2.0 ** (ns - args.n),
            "digest": r["digest"], "stages": r["stages"]}


def sample_text(args, s, cores) -> str:
    return (f"{args.circuit}-{s['n_sample']} full circuit ({s['gates']} gates, c={args.c} "
            f"m={min(args.m, s['n_sample'])} eb={args.eb}, {s['stages']} stages) through the "
            f"unmodified reference qzsim::run with {cores} decompress/recompress/kernel workers, "
            f"{s['wall_seconds']:.2f} s = {s['gates_per_s_sample']:.2f} gates/s, scaled by "
            f"2^({s['n_sample']}-{args.n}) to n={args.n}; host {cpu_info()}")


def cpu_info() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args, gates):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    cfg = workload_config(args)
    vals, samples = [], []
    first = reference_sample(args.circuit, args.n, args.c, args.m, args.eb, args.cpu_budget)
    for i in range(args.warmup + args.steps):
        s = first if i == 0 else reference_sample_fixed(args, first)
        if i >= args.warmup:
            vals.append(s["gates_per_s"])
            samples.append(s)
    v = statistics.median(vals)
    s = samples[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "gates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * s["wall_seconds"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": v, "unit": "gates/s", "cores": cores, "kind": "reference",
                         "sample": sample_text(args, s, cores)},
        "e2e": {"value": v, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_config(args) -> dict:
    where = "HBM-resident store" if args.residency == "hbm" else "host-staged store (pinned host RAM)"
    return {"workload": f"{args.circuit}-{args.n} compressed-chunk pipeline, {where}",
            "circuit": args.circuit, "num_qubits": args.n, "chunk_qubits": args.c,
            "batch_qubits": args.m, "error_bound": args.eb,
            "l2": "inputs larger than L2 (2^n x 16 B dense state per stage sweep)"}


# ----------------------------------------------------------------- engine --
def main() -> int:
    args = parse_args()
    from paper_2309_16979_b200 import circuits
    gates = circuits.make(args.circuit, args.n)
    if args.impl == "reference":
        return run_reference_arm(args, gates)

    from paper_2309_16979_b200.engine import Engine
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    eng = Engine(device=local)
    ngates = len(gates)
    if args.shard and world > 1:
        return run_sharded(args, eng, gates, dist, rank, world, local)
    sim = eng.simulator(args.n, args.c, args.m, args.eb, init=False,
                        fuse=False if args.no_fuse else ("strict" if args.strict_passes else True),
                        residency=args.residency)

    for _ in range(args.warmup):
        sim.init_basis()
        sim.run(gates)

    # ---- timed region: K steps, device time (CUDA events on the engine stream)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(1.0)   # nvidia-smi's first samples arrive before the timed region
    barrier()
    eng.timer_begin()
    eng.timer_end()
    launches0 = eng.kernel_launches
    clocks.mark_begin()
    eng.timer_begin()
    for _ in range(args.steps):
        sim.init_basis()
        sim.run(gates)
    t_dev = eng.timer_end()
    clocks.mark_end()
    launches = eng.kernel_launches - launches0
    clk = clocks.stop()
    t_max = max_over_ranks(t_dev)
    barrier()
    st = sim.stats()          # last step's counters
    digest = sim.digest()

    # ---- end to end through the public API: host gate list in, host store out
    e2e_times = []
    h2d = gates.nbytes
    d2h = 0
    # page-locked result buffers, allocated once like a serving loop's
    cap = sim.payload_bytes() * 5 // 4 + (1 << 20)
    out = eng.pinned(cap)
    out_sizes = eng.pinned(4 * sim.chunk_count, np.uint32)
    out_crcs = eng.pinned(4 * sim.chunk_count, np.uint32)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        eng.timer_begin()
        sim.init_basis()
        sim.run(gates)
        blob, sizes, crcs = sim.export(out, out_sizes, out_crcs)
        eng.timer_end()
        e2e_times.append(time.perf_counter() - t0)
        d2h = len(blob) + sizes.nbytes + crcs.nbytes
    e2e_t = max_over_ranks(statistics.median(e2e_times))

    if rank != 0:
        return 0

    # ---- fidelity of the compressed run against an uncompressed fp64 run of
    # the same circuit on the GPU (outside the timed region; BASELINE metric)
    fidelity = None
    if not args.no_fidelity:
        try:
            dense = eng.dense_state(args.n, gates)
            fidelity = sim.fidelity(dense)
            dense.free()
        except Exception as e:  # not enough HBM for the dense state next to the store
            fidelity = f"unavailable: {e}"

    value = world * ngates * args.steps / t_max
    # ---- roofline of the dominant kernel (from the engine's event timers)
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    phases = {"decode": st["decode_seconds"], "gates": st["gate_seconds"],
              "encode": st["encode_seconds"]}
    win_amps = (1 << args.n) // max(1, st["windows"] // max(1, st["stages"]))
    pass_bytes = 32 * win_amps
    avg_pass = st["gate_seconds"] / max(1, st["gate_passes"])
    gate_ach = pass_bytes / avg_pass / 1e9 if avg_pass > 0 else 0.0
    payload = len(blob)
    dec_bytes = st["stages"] * (16 * (1 << args.n) + payload)   # approx: final payload size
    enc_bytes = dec_bytes
    # measured DRAM bytes per launch of the dominant kernel from the committed
    # `ncu --set full` capture (profiles/traffic.json, written by
    # tools/profile_round.sh) for this workload, when present
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        t = json.loads(tfile.read_text()).get(f"{args.circuit}-{args.n}-m{args.m}")
        traffic = t["dram_bytes_per_launch"] if t else None
    roofline = {"bound": "hbm", "kernel": "tile_pass_reg + tile_swaps (fused gate passes)",
                "achieved": gate_ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": gate_ach / hbm_peak, "traffic": traffic,
                "bytes_per_launch": pass_bytes, "avg_launch_s": avg_pass,
                "launches": st["gate_passes"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                "codec": {"decode_GBps": dec_bytes / st["decode_seconds"] / 1e9 if st["decode_seconds"] else None,
                          "encode_GBps": enc_bytes / st["encode_seconds"] / 1e9 if st["encode_seconds"] else None,
                          "note": "decode/encode phase = crc+index+decode / encode+size+scan+assemble+crc"}}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            s = reference_sample(args.circuit, args.n, args.c, args.m, args.eb, args.cpu_budget)
            cpu = {"value": s["gates_per_s"], "unit": "gates/s", "cores": os.cpu_count(),
                   "kind": "reference", "sample": sample_text(args, s, os.cpu_count())}
        except Exception as e:  # reference library absent on this box
            cpu = {"value": None, "unit": "gates/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    host_link = None
    if args.residency == "host":
        link = eng.host_link_gbps()
        io = st["h2d_bytes"] + st["d2h_bytes"]
        ach = io / (t_max / args.steps) / 1e9
        host_link = {"bound": "host-link", "achieved": ach, "unit": "GB/s",
                     "h2d_peak": link["h2d"], "d2h_peak": link["d2h"],
                     "frac": ach / max(link["h2d"], link["d2h"]),
                     "bytes_per_step": io,
                     "note": "compressed payload bytes moved host<->HBM per circuit / circuit "
                             "time, vs measured pinned cudaMemcpy bandwidth"}
    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": dict(workload_config(args), parallelism=f"replicas{world}",
                                            gates=ngates),
        "circuit_seconds": t_max / args.steps,
        "compression_ratio": st["ratio"],
        "fidelity": fidelity,
        "peak_ratio": st["dense_bytes"] / st["peak_bytes"] if st["peak_bytes"] else None,
        "digest": f"{digest:016x}",
        "phases_s": phases, "stages": st["stages"], "gate_passes": st["gate_passes"],
        "replays": st["replays"],
        "gpu_launches": launches,
        "roofline": roofline,
        "host_link": host_link,
        "cpu_baseline": cpu,
        "e2e": {"value": world * ngates / e2e_t, "unit": "gates/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "clocks": clk,
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def run_sharded(args, eng, gates, dist, rank, world, local):
    """One circuit over all ranks (sharding.py): each rank owns 2^(n-c-g)
    chunks; compressed chunks move over NCCL at ownership changes."""
    import torch
    from paper_2309_16979_b200 import sharding as S
    g = world.bit_length() - 1
    if 1 << g != world:
        raise SystemExit("--shard needs a power-of-two number of ranks")
    grp = S.TorchGroup(dist, device=f"cuda:{local}")
    run = S.ShardedRun(eng, args.n, args.c, args.m, args.eb, g, [rank], grp)
    for _ in range(args.warmup):
        run.owners = list(range(args.n - g, args.n))
        run.init_basis()
        run.run(gates)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ex0 = run.exchanged_bytes
    for _ in range(args.steps):
        run.owners = list(range(args.n - g, args.n))
        run.init_basis()
        run.run(gates)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    digest = run.digest()
    if rank == 0:
        tmax = float(t.item())
        print(json.dumps({
            "metric": METRIC, "value": len(gates) * args.steps / tmax, "unit": "gates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tmax / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(args), parallelism=f"shard{world}", gates=len(gates)),
            "digest": f"{digest:016x}", "exchanges": run.exchanges,
            "exchanged_bytes_per_step": (run.exchanged_bytes - ex0) // max(1, args.steps),
            "timing": "device-synchronized interval, max over ranks"}))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
