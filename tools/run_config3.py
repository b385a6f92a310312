"""SURVEY cfg3: supremacy-style depth-20 circuit at n qubits with the
compressed store host-staged (mapped page-locked host arenas, HBM windows).
One run from |0...0>, CUDA-event timed on the engine stream; prints one JSON
line with throughput, compression, stage / transfer counts and the host-link
roofline."""
import argparse
import json
import time

from paper_2309_16979_b200 import circuits
from paper_2309_16979_b200.engine import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=34)
ap.add_argument("--c", type=int, default=16)
ap.add_argument("--m", type=int, default=30)
ap.add_argument("--eb", type=float, default=1e-7)
ap.add_argument("--depth", type=int, default=20)
ap.add_argument("--residency", default="host")
a = ap.parse_args()

eng = Engine()
gates = circuits.supremacy(a.n, depth=a.depth)
link = eng.host_link_gbps(1 << 30, 3)
t0 = time.perf_counter()
sim = eng.simulator(a.n, a.c, a.m, a.eb, residency=a.residency, init=False)
t1 = time.perf_counter()
eng.timer_begin()
sim.init_basis()
sim.run(gates)
t_dev = eng.timer_end()
t2 = time.perf_counter()
st = sim.stats()
io = st["h2d_bytes"] + st["d2h_bytes"]
print(json.dumps({
    "workload": f"supremacy-{a.n} depth {a.depth}, c={a.c} m={a.m} eb={a.eb}, {a.residency}-resident store",
    "gates": len(gates), "seconds": t_dev, "gates_per_s": len(gates) / t_dev,
    "amp_gate_updates_per_s": len(gates) * 2.0 ** a.n / t_dev,
    "setup_seconds": t1 - t0, "wall_seconds": t2 - t1,
    "stages": st["stages"], "windows": st["windows"], "gate_passes": st["gate_passes"],
    "replays": st["replays"], "phases_s": {"decode": st["decode_seconds"], "gates": st["gate_seconds"],
                                           "encode": st["encode_seconds"]},
    "compression_ratio": st["ratio"], "current_bytes": st["current_bytes"], "peak_bytes": st["peak_bytes"],
    "dense_bytes": st["dense_bytes"], "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"],
    "host_link": {"achieved_GBps": io / t_dev / 1e9, "h2d_peak_GBps": link["h2d"], "d2h_peak_GBps": link["d2h"]},
}))
