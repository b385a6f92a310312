#!/usr/bin/env python3
"""bench.py — MEMQSim hot path on B200: gates/s and circuit time at n qubits.

Default workload (BASELINE.json configs[1]): 30-qubit QFT (2220 gates) from
|0...0>, compressed-chunk store fully resident in HBM, c=16, m=30, eb=1e-5.
A step = one circuit execution through the staged pipeline: store init
(store.cpp:26-81) + every stage's decode → fused gate passes → encode
(pipeline.cpp:128-314), ending with the final compressed store in HBM.

  python bench.py [--gpus N --steps K --warmup W]          engine arm
  python bench.py --impl reference [...]                   reference CPU arm

Roofline: every engine kernel launch inside the timed region is bracketed by
CUDA events on its own stream (qzc_kprof_*); `roofline` is the DOMINANT
launch (largest share of the step) with its algorithmic bytes (SURVEY §8d:
32 B per window amplitude for a gate pass), and `roofline.kernels` lists
every kernel family (codec families with their payload bytes added).

Companions (N=1, extra key `companions`): dense workloads the headline QFT
does not exercise — supremacy-30 depth 20 at eb=1e-7 (codec on dense
chunks, fidelity < 1) and QFT-30 at m=20 (37 stages, codec-dominated).

Multi-GPU (torchrun, one rank per GPU; `--gpus N` without torchrun
re-launches itself under torchrun): `--mode shard` (default for N>1) runs
ONE circuit over all ranks with compressed chunks exchanged device to
device over NCCL at ownership changes (strong scaling); `--mode replicas`
runs an independent replica per rank (weak scaling).
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
FALLBACK_HBM = 6650.0   # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def parse_args(argv=None):
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
    ap.add_argument("--depth", type=int, default=20, help="supremacy depth")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fidelity", action="store_true",
                    help="skip the uncompressed fp64 reference run used for the fidelity figure")
    ap.add_argument("--no-companions", action="store_true")
    ap.add_argument("--companion-cpu", action="store_true",
                    help="also time the reference on the companions (2 x ~1 min each at n=30)")
    ap.add_argument("--no-kprof", action="store_true",
                    help="no per-launch events in the timed region (roofline from phase totals)")
    ap.add_argument("--fuse", default="relaxed", choices=["relaxed", "strict", "checked", "none"])
    ap.add_argument("--mode", default=None, choices=["shard", "replicas"],
                    help="N>1: shard one circuit over the ranks (default) or run replicas")
    ap.add_argument("--residency", default="hbm", choices=["hbm", "host"],
                    help="compressed store in HBM (config 2) or pinned host memory (config 3)")
    return ap.parse_args(argv)


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
def cpu_info() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def make_circuit(name: str, n: int, depth: int = 20):
    from paper_2309_16979_b200 import circuits
    if name == "supremacy":
        return circuits.supremacy(n, depth=depth)
    return circuits.make(name, n)


def prefix_lengths(name: str, n: int) -> tuple[int, int]:
    """Two gate-prefix lengths of the circuit for the reference sample, 40
    gates apart so the per-gate cost (~0.3 s per gate at n=30 on 16 cores)
    stands well above the run-to-run noise of the stage sweep: the first
    Hadamard, then it plus 8 controlled-phase blocks for the QFT; 1 and 41
    gates otherwise."""
    if name == "qft":
        return 1, 41
    return 1, 41


class ReferenceSampler:
    """The UNMODIFIED reference qzsim::run (oracle/_ref/libqzref.so) on a
    bounded sample of the SAME workload: the circuit's first k1 and k2 gates
    at the full n, c, m and eb, on every host core.  Its own report
    wall_seconds (pipeline.cpp:158-290) is T(k) = T0 + k * t_gate (T0 =
    init + one codec sweep of the 2^n state, t_gate = one reference gate
    pass over 2^n amplitudes), so the full circuit's time is estimated as
    T(k1) + (G - k1) * (T(k2) - T(k1)) / (k2 - k1)."""

    def __init__(self, args):
        sys.path.insert(0, str(ROOT / "tests"))
        from oracles import Reference  # baseline infrastructure only
        self.ref = Reference()
        self.args = args
        self.gates = make_circuit(args.circuit, args.n, args.depth)
        self.k1, self.k2 = prefix_lengths(args.circuit, args.n)
        self.times = {self.k1: [], self.k2: []}
        self.cores = os.cpu_count() or 1

    def sample(self, k: int) -> float:
        a = self.args
        # Synchronous strategy: the reference's device bound is 2^m x 16 B
        # instead of twice that (results are strategy-invariant)
        r = self.ref.run(a.n, self.gates[:k], a.c, min(a.m, a.n), a.eb, workers=0, depth=2,
                         strategy=0)
        self.times[k].append(r["wall_seconds"])
        return r["wall_seconds"]

    def estimate(self) -> dict:
        from paper_2309_16979_b200.sharding import global_stages
        a = self.args
        t1 = statistics.median(self.times[self.k1])
        t2 = statistics.median(self.times[self.k2])
        per_gate = max((t2 - t1) / (self.k2 - self.k1), 1e-9)
        g = len(self.gates)
        # both prefixes are one stage; every further stage adds one codec
        # sweep T0 = T(k1) - k1 * per_gate (pipeline.cpp:159-276)
        self.stages = len(global_stages(a.n, a.c, min(a.m, a.n), self.gates))
        t0 = max(t1 - self.k1 * per_gate, 0.0)
        full = self.stages * t0 + g * per_gate
        return {"t_k1": t1, "t_k2": t2, "per_gate_s": per_gate, "sweep_s": t0,
                "stages": self.stages, "full_circuit_s": full, "gates_per_s": g / full}

    def text(self, est) -> str:
        a = self.args
        return (f"{a.circuit}-{a.n} (c={a.c} m={a.m} eb={a.eb}, the engine arm's config): the "
                f"unmodified reference qzsim::run on its first {self.k1} and {self.k2} gates with "
                f"{self.cores} decompress/recompress/kernel workers (Synchronous strategy), "
                f"{est['t_k1']:.2f} s / {est['t_k2']:.2f} s -> {est['per_gate_s']:.3f} s per gate, "
                f"{est['sweep_s']:.2f} s per stage sweep; full {len(self.gates)}-gate circuit "
                f"({est['stages']} stages) estimated at {est['full_circuit_s']:.1f} s "
                f"(stages x sweep + G x per-gate); host {cpu_info()}")


def run_reference_arm(args) -> int:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    s = ReferenceSampler(args)
    ks = [s.k1, s.k2]
    # warm-up: the reference's thread pools and code paths on a small
    # instance of the same circuit family (a CPU library has no JIT or
    # cache state worth a full 2^n sweep per warm-up step)
    warm = argparse.Namespace(**vars(args))
    warm.n = min(args.n, max(args.c + 2, 20))
    warm.m = min(args.m, warm.n)
    ws = ReferenceSampler(warm)
    for i in range(args.warmup):
        ws.sample(ks[i % 2])
    # each step is one full-size sample (~1 min at n=30 on 16 cores): the two
    # the estimate needs, then more only while the run stays within a few
    # minutes (QZ_REF_BUDGET_S, default 240 s); "steps" reports those done
    budget = float(os.environ.get("QZ_REF_BUDGET_S", "240"))
    walls = []
    t_start = time.perf_counter()
    for i in range(max(args.steps, 2)):
        if i >= 2 and time.perf_counter() - t_start > budget:
            break
        t0 = time.perf_counter()
        s.sample(ks[i % 2])
        walls.append(time.perf_counter() - t0)
    est = s.estimate()
    v = est["gates_per_s"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "gates/s",
        "n_gpus": args.gpus, "steps": len(walls), "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(walls), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": "gates/s", "cores": s.cores, "kind": "reference",
                         "sample": s.text(est)},
        "reference_samples_s": {str(k): v for k, v in s.times.items()},
        "full_circuit_s_estimate": est["full_circuit_s"],
        "step": "one run of the circuit's first k1 or k2 gates (alternating) at the full "
                "n, c, m, eb; value = gates / (stages x sweep + gates x per-gate) from them",
        "e2e": {"value": v, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_config(args, circuit=None, n=None, m=None, eb=None) -> dict:
    circuit = circuit or args.circuit
    n = n or args.n
    m = m or args.m
    eb = eb or args.eb
    where = "HBM-resident store" if args.residency == "hbm" else "host-staged store (pinned host RAM)"
    cfg = {"workload": f"{circuit}-{n} compressed-chunk pipeline, {where}",
           "circuit": circuit, "num_qubits": n, "chunk_qubits": args.c,
           "batch_qubits": m, "error_bound": eb,
           "l2": "inputs larger than L2 (2^n x 16 B dense state per stage sweep)"}
    if circuit == "supremacy":
        cfg["depth"] = args.depth
    return cfg


# ----------------------------------------------------------------- engine --
def peaks() -> tuple[float, str]:
    if PEAKS.exists():
        p = json.loads(PEAKS.read_text())
        if p.get("hbm_gbs"):
            return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy read+write, burst)"
    return FALLBACK_HBM, "B200_PROFILING.md fallback"


def family(name: str) -> str:
    if name.startswith(("tile_pass_reg", "tile_pass_jit")):
        return "gate_pass"
    if name == "tile_swaps":
        return "swap_pass"
    if name in ("k_dec_lossy_seg", "k_dec_lossy_warp", "k_dec_lossy", "k_dec_lossless"):
        return "decode"
    if name in ("k_enc_lossy", "k_enc_lossy_direct", "k_enc_lossless"):
        return "encode"
    return name


def roofline_from_kprof(recs, steps, stats, hbm_peak, peak_src) -> dict:
    """Dominant launch (largest share of the step) + per-family rooflines.
    Records of the timed region only; a launch is keyed by (stage, kernel,
    pass index) so the same pass of every step averages together."""
    run = [r for r in recs if r["stage"] != 0xFFFFFFFF]
    per_key = {}
    for r in run:
        per_key.setdefault((r["stage"], r["name"], r["tag"]), []).append(r)
    total = sum(r["seconds"] for r in run) / steps
    best, best_t = None, -1.0
    for key, rs in per_key.items():
        if key[1] in ("replay_pass", "replay_decode"):
            continue
        t = sum(r["seconds"] for r in rs) / steps
        if t > best_t:
            best, best_t = key, t
    rs = per_key[best]
    avg = sum(r["seconds"] for r in rs) / len(rs)
    nbytes = rs[0]["bytes"]
    fam = {}
    for r in recs:   # init_basis included in the families (its kernels run in the step)
        f = fam.setdefault(family(r["name"]), {"seconds": 0.0, "bytes": 0.0, "launches": 0})
        f["seconds"] += r["seconds"] / steps
        f["bytes"] += r["bytes"] / steps
        f["launches"] += 1
    # codec families: compressed bytes read / written per step (stats are the last step's)
    if "decode" in fam:
        fam["decode"]["bytes"] += stats["payload_in_bytes"]
    if "encode" in fam:
        fam["encode"]["bytes"] += stats["payload_out_bytes"]
    kernels = {}
    for k, f in sorted(fam.items(), key=lambda kv: -kv[1]["seconds"]):
        ach = f["bytes"] / f["seconds"] / 1e9 if f["seconds"] > 0 and f["bytes"] > 0 else None
        kernels[k] = {"ms_per_step": 1e3 * f["seconds"], "share": f["seconds"] / total if total else None,
                      "launches_per_step": f["launches"] / steps,
                      "GBps": ach, "frac": ach / hbm_peak if ach else None}
    ach = nbytes / avg / 1e9
    return {"bound": "hbm", "kernel": f"{best[1]} (stage {best[0]}, pass {best[2]})",
            "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "traffic": None, "bytes_per_launch": nbytes, "avg_launch_s": avg,
            "share_of_step": best_t / total if total else None,
            "peak_source": peak_src,
            "bytes_basis": "algorithmic: 32 B per window amplitude per gate pass (read + write), "
                           "codec families 16 B per dense amplitude + compressed payload bytes",
            "kernels": kernels}


def committed_traffic(key: str, kernel: str):
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        t = json.loads(tfile.read_text()).get(key)
        if t and t.get("kernel", kernel).split(" ")[0] == kernel.split(" ")[0]:
            return t
    return None


def timed_steps(eng, sim, gates, steps, local, kprof=True):
    """K steps of init + run on the device clock; returns (seconds, kprof
    records, clocks, engine launches)."""
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(1.0)   # nvidia-smi's first samples arrive before the timed region
    eng.timer_begin()
    eng.timer_end()
    launches0 = eng.kernel_launches
    if kprof:
        eng.kprof_enable(True)
    clocks.mark_begin()
    eng.timer_begin()
    for _ in range(steps):
        sim.init_basis()
        sim.run(gates)
    t_dev = eng.timer_end()
    clocks.mark_end()
    recs = eng.kprof_read() if kprof else []
    eng.kprof_enable(False)
    launches = eng.kernel_launches - launches0
    return t_dev, recs, clocks.stop(), launches


def fidelity_of(eng, sim, n, gates):
    try:
        dense = eng.dense_state(n, gates)
        f = sim.fidelity(dense)
        dense.free()
        return {"fidelity": f, "infidelity": 1.0 - f}
    except Exception as e:  # not enough HBM for the dense state next to the store
        return {"fidelity": None, "infidelity": None, "note": f"unavailable: {e}"}


def warmup_steps(step, warmup: int) -> dict:
    """W untimed steps.  After the first, wait for the runtime-specialised
    gate passes it queued (NVRTC on host threads, qz_jit.cu) so the timed
    steps run the kernels a long job runs; one-time compile cost reported."""
    from paper_2309_16979_b200.engine import jit_wait
    step()
    t0 = time.perf_counter()
    built = jit_wait()
    wait = time.perf_counter() - t0
    for _ in range(max(warmup - 1, 1)):
        step()
    return {"specialised_passes": built, "jit_wait_s": round(wait, 2)}


def companion(eng, args, name, n, m, eb, depth, steps, warmup, hbm_peak, peak_src, cpu=True,
              skip_reencode=False):
    """A second workload timed the same way (extra key, not the headline).
    skip_reencode: the NON-PARITY fast mode (one stage when the state fits)."""
    from paper_2309_16979_b200 import circuits
    gates = circuits.supremacy(n, depth=depth) if name == "supremacy" else circuits.make(name, n)
    sim = eng.simulator(n, args.c, m, eb, init=False, skip_reencode=skip_reencode)
    def step():
        sim.init_basis()
        sim.run(gates)
    jit = warmup_steps(step, warmup)
    t, recs, clk, launches = timed_steps(eng, sim, gates, steps, eng.device)
    st = sim.stats()
    out = {"workload": f"{name}-{n}" + (f" depth {depth}" if name == "supremacy" else "") +
                       f" c={args.c} m={m} eb={eb}, HBM-resident" +
                       (", NON-PARITY skip-reencode mode (one stage per run)" if skip_reencode else ""),
           "parity": not skip_reencode,
           "gates": len(gates), "value": len(gates) * steps / t, "unit": "gates/s",
           "ms_per_step": 1e3 * t / steps, "steps": steps, "stages": st["stages"],
           "gate_passes": st["gate_passes"], "replays": st["replays"],
           "compression_ratio": st["ratio"], "digest": f"{sim.digest():016x}",
           "phases_ms": {"decode": 1e3 * st["decode_seconds"], "gates": 1e3 * st["gate_seconds"],
                         "encode": 1e3 * st["encode_seconds"]},
           "payload_in_GB": st["payload_in_bytes"] / 1e9, "payload_out_GB": st["payload_out_bytes"] / 1e9,
           "gpu_launches": launches, "clocks": clk, **jit}
    out["roofline"] = roofline_from_kprof(recs, steps, st, hbm_peak, peak_src)
    out.update(fidelity_of(eng, sim, n, gates))
    sim.close()
    if cpu:
        try:
            a = argparse.Namespace(**vars(args))
            a.circuit, a.n, a.m, a.eb, a.depth = name, n, m, eb, depth
            s = ReferenceSampler(a)
            for k in (s.k1, s.k2):
                s.sample(k)
            est = s.estimate()
            out["cpu_baseline"] = {"value": est["gates_per_s"], "unit": "gates/s", "cores": s.cores,
                                   "kind": "reference", "sample": s.text(est)}
        except Exception as e:
            out["cpu_baseline"] = {"value": None, "sample": f"unavailable: {e}"}
    return out


def relaunch_under_torchrun(args) -> int:
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main() -> int:
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    gates = make_circuit(args.circuit, args.n, args.depth)

    from paper_2309_16979_b200.engine import Engine
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    mode = args.mode or ("shard" if world > 1 else "replicas")
    eng = Engine(device=local)
    if world > 1 and mode == "shard":
        return run_sharded(args, eng, gates, dist, rank, world, local)

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

    ngates = len(gates)
    fuse = {"relaxed": True, "strict": "strict", "checked": "checked", "none": False}[args.fuse]
    sim = eng.simulator(args.n, args.c, args.m, args.eb, init=False, fuse=fuse,
                        residency=args.residency)
    def step():
        sim.init_basis()
        sim.run(gates)
    jit = warmup_steps(step, args.warmup)

    # ---- timed region: K steps, device time (CUDA events on the engine stream)
    barrier()
    t_dev, recs, clk, launches = timed_steps(eng, sim, gates, args.steps, local,
                                             kprof=not args.no_kprof)
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
        if dist:
            dist.destroy_process_group()
        return 0

    hbm_peak, peak_src = peaks()
    value = world * ngates * args.steps / t_max
    fid = {"fidelity": None, "infidelity": None} if args.no_fidelity else \
        fidelity_of(eng, sim, args.n, gates)
    if recs:
        roofline = roofline_from_kprof(recs, args.steps, st, hbm_peak, peak_src)
        tr = committed_traffic(f"{args.circuit}-{args.n}-m{args.m}", roofline["kernel"])
        if tr:
            roofline["traffic"] = tr["dram_bytes_per_launch"]
            roofline["traffic_source"] = tr.get("source", "profiles/traffic.json")
    else:
        roofline = {"bound": "hbm", "note": "--no-kprof: no per-launch timing"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            s = ReferenceSampler(args)
            for k in (s.k1, s.k2):
                s.sample(k)
            est = s.estimate()
            cpu = {"value": est["gates_per_s"], "unit": "gates/s", "cores": s.cores,
                   "kind": "reference", "sample": s.text(est)}
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

    companions = []
    if world == 1 and not args.no_companions and args.circuit == "qft" and args.n == 30:
        sim.close()
        for (name, n, m, eb, depth, steps, fast) in (("supremacy", 30, 30, 1e-7, 20, 2, False),
                                                     ("qft", 30, 20, 1e-5, 20, 2, False),
                                                     ("qft", 30, 20, 1e-5, 20, 2, True)):
            try:
                companions.append(companion(eng, args, name, n, m, eb, depth, steps, 1, hbm_peak,
                                            peak_src, cpu=args.companion_cpu and not fast,
                                            skip_reencode=fast))
            except Exception as e:
                companions.append({"workload": f"{name}-{n} m={m}", "error": str(e)})

    line = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": dict(workload_config(args), parallelism=f"replicas{world}",
                                            gates=ngates, **jit),
        "circuit_seconds": t_max / args.steps,
        "compression_ratio": st["ratio"],
        "fidelity": fid["fidelity"], "infidelity": fid["infidelity"],
        "peak_ratio": st["dense_bytes"] / st["peak_bytes"] if st["peak_bytes"] else None,
        "digest": f"{digest:016x}",
        "phases_s": {"decode": st["decode_seconds"], "gates": st["gate_seconds"],
                     "encode": st["encode_seconds"]},
        "stages": st["stages"], "gate_passes": st["gate_passes"], "replays": st["replays"],
        "gpu_launches": launches,
        "roofline": roofline,
        "host_link": host_link,
        "cpu_baseline": cpu,
        "e2e": {"value": world * ngates / e2e_t, "unit": "gates/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "clocks": clk,
        "companions": companions,
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def run_sharded(args, eng, gates, dist, rank, world, local):
    """One circuit over all ranks (sharding.py): each rank owns 2^(n-c-g)
    chunks; compressed chunks move device to device over NCCL at ownership
    changes.  Strong scaling: the total work is fixed as N grows."""
    import torch
    from paper_2309_16979_b200 import sharding as S
    g = world.bit_length() - 1
    if 1 << g != world:
        raise SystemExit("--mode shard needs a power-of-two number of ranks")
    grp = S.TorchGroup(dist, device=f"cuda:{local}")
    # each rank's local register has n - g qubits: the batch window shrinks to fit
    m = min(args.m, args.n - g)
    run = S.ShardedRun(eng, args.n, args.c, m, args.eb, g, [rank], grp)
    def step():
        run.init_basis()
        run.run(gates)
    jit = warmup_steps(step, args.warmup)
    dist.barrier()
    torch.cuda.synchronize()
    ex0, b0 = run.exchanges, run.exchanged_bytes
    eng.timer_begin()
    for _ in range(args.steps):
        run.init_basis()
        run.run(gates)
    el = eng.timer_end()
    t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tmax = float(t.item())
    # e2e: the same through the public API with the sharded store gathered
    # to host memory at the end of every step
    e2e = []
    d2h = 0
    for _ in range(max(1, args.steps // 2)):
        dist.barrier()
        t0 = time.perf_counter()
        run.init_basis()
        run.run(gates)
        d2h = sum(len(blob) + sizes.nbytes + crcs.nbytes for blob, sizes, crcs in run.local_export().values())
        dist.barrier()
        e2e.append(time.perf_counter() - t0)
    te = torch.tensor([statistics.median(e2e)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    digest = run.digest()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": len(gates) * args.steps / tmax, "unit": "gates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tmax / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(args, m=m), parallelism=f"shard{world}", gates=len(gates),
                           transport="NCCL send/recv of compressed chunk records, device to device", **jit),
            "digest": f"{digest:016x}", "exchanges_per_step": (run.exchanges - ex0) / args.steps,
            "exchanged_bytes_per_step": (run.exchanged_bytes - b0) // max(1, args.steps),
            "gpu_launches": eng.kernel_launches,
            "e2e": {"value": len(gates) / float(te.item()), "unit": "gates/s",
                    "h2d_bytes_per_step": int(gates.nbytes), "d2h_bytes_per_step": int(d2h) * world},
            "timing": "CUDA events on the engine stream, max over ranks"}))
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
