"""Large single-GPU runs (SURVEY cfg3 and the qubit-ceiling row): one circuit
at n qubits from |0...0>, compressed store HBM-resident or host-staged,
CUDA-event timed on the engine stream, SM clocks sampled by nvidia-smi
during the run (bench.ClockSampler), per-kernel event totals, one JSON line.

  python tools/run_large.py --circuit supremacy --n 34 --residency host
  python tools/run_large.py --circuit qft --n 36 --m 30 --eb 1e-5
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import ClockSampler  # noqa: E402
from paper_2309_16979_b200 import circuits  # noqa: E402
from paper_2309_16979_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--circuit", default="supremacy")
ap.add_argument("--n", type=int, default=34)
ap.add_argument("--c", type=int, default=16)
ap.add_argument("--m", type=int, default=30)
ap.add_argument("--eb", type=float, default=1e-7)
ap.add_argument("--depth", type=int, default=20)
ap.add_argument("--residency", default="host", choices=["host", "hbm"])
ap.add_argument("--window", type=int, default=0, help="window amplitudes (0 = auto)")
a = ap.parse_args()

eng = Engine()
gates = circuits.supremacy(a.n, depth=a.depth) if a.circuit == "supremacy" else circuits.make(a.circuit, a.n)
link = eng.host_link_gbps(1 << 30, 3) if a.residency == "host" else None
t0 = time.perf_counter()
sim = eng.simulator(a.n, a.c, a.m, a.eb, residency=a.residency, init=False, window_amps=a.window)
t1 = time.perf_counter()
clk = ClockSampler(0)
clk.start()
time.sleep(1.0)
eng.kprof_enable(True)
clk.mark_begin()
eng.timer_begin()
sim.init_basis()
sim.run(gates)
t_dev = eng.timer_end()
clk.mark_end()
t2 = time.perf_counter()
kernels = {}
for r in eng.kprof_read():
    k = kernels.setdefault(r["name"], {"launches": 0, "seconds": 0.0})
    k["launches"] += 1
    k["seconds"] += r["seconds"]
eng.kprof_enable(False)
clocks = clk.stop()
st = sim.stats()
io = st["h2d_bytes"] + st["d2h_bytes"]
out = {
    "workload": f"{a.circuit}-{a.n}" + (f" depth {a.depth}" if a.circuit == "supremacy" else "") +
                f", c={a.c} m={a.m} eb={a.eb}, {a.residency}-resident store",
    "gates": len(gates), "seconds": t_dev, "gates_per_s": len(gates) / t_dev,
    "amp_gate_updates_per_s": len(gates) * 2.0 ** a.n / t_dev,
    "dense_state_GB": 16 * 2 ** a.n / 1e9,
    "setup_seconds": t1 - t0, "wall_seconds": t2 - t1,
    "stages": st["stages"], "windows": st["windows"], "gate_passes": st["gate_passes"],
    "replays": st["replays"], "phases_s": {"decode": st["decode_seconds"], "gates": st["gate_seconds"],
                                           "encode": st["encode_seconds"]},
    "compression_ratio": st["ratio"], "current_bytes": st["current_bytes"], "peak_bytes": st["peak_bytes"],
    "dense_bytes": st["dense_bytes"], "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"],
    "kernels_s": {k: round(v["seconds"], 4) for k, v in sorted(kernels.items(), key=lambda kv: -kv[1]["seconds"])},
    "kernel_times_note": "per-launch CUDA events; launches of concurrent window streams overlap",
    "clocks": clocks,
}
if link:
    out["host_link"] = {"achieved_GBps": io / t_dev / 1e9, "h2d_peak_GBps": link["h2d"],
                        "d2h_peak_GBps": link["d2h"],
                        "frac": io / t_dev / 1e9 / (link["h2d"] + link["d2h"]),
                        "note": "H2D + D2H compressed payload bytes over both link directions' peaks"}
print(json.dumps(out), flush=True)
