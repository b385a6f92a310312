"""Dense-state codec / pass timing probe: one circuit at n qubits, per-phase
CUDA-event times and the store size (the codec's dense-workload numbers)."""
import argparse
import time

from paper_2309_16979_b200 import circuits
from paper_2309_16979_b200.engine import Engine, jit_wait

ap = argparse.ArgumentParser()
ap.add_argument("circuit")
ap.add_argument("n", type=int)
ap.add_argument("--c", type=int, default=16)
ap.add_argument("--m", type=int, default=30)
ap.add_argument("--eb", type=float, default=1e-7)
ap.add_argument("--depth", type=int, default=20)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kprof", action="store_true", help="per-kernel CUDA-event totals of the last rep")
a = ap.parse_args()
eng = Engine()
kw = {"depth": a.depth} if a.circuit == "supremacy" else {}
gates = circuits.make(a.circuit, a.n, **kw)
sim = eng.simulator(a.n, a.c, a.m, a.eb, init=False)
for rep in range(a.reps):
    if a.kprof and rep == a.reps - 1:
        eng.kprof_enable(True)
    t0 = time.perf_counter()
    sim.init_basis()
    sim.run(gates)
    st = sim.stats()
    el = time.perf_counter() - t0
    print(f"{a.circuit}-{a.n} c={a.c} m={a.m} eb={a.eb}: {1e3*el:.1f} ms, stages {st['stages']} "
          f"windows {st['windows']} passes {st['gate_passes']} replays {st['replays']} "
          f"dec {1e3*st['decode_seconds']:.2f} gates {1e3*st['gate_seconds']:.2f} "
          f"enc {1e3*st['encode_seconds']:.2f} ms payload {sim.payload_bytes()/1e9:.3f} GB "
          f"ratio {st['ratio']:.3f} digest {sim.digest():016x}", flush=True)
    if rep == 0:
        t0 = time.perf_counter()
        built = jit_wait()
        print(f"  specialised passes built: {built} (waited {time.perf_counter() - t0:.1f} s)", flush=True)
if a.kprof:
    tot = {}
    for r in eng.kprof_read():
        k = r["name"] + (f" #{r['tag']}" if r["name"].startswith("tile") and r["stage"] == 0 else "")
        t = tot.setdefault(k, [0, 0.0, 0.0])
        t[0] += 1
        t[1] += r["seconds"]
        t[2] += r["bytes"]
    for k, (n, sec, b) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:24s} launches {n:5d}  {1e3*sec:9.2f} ms  dense {b/1e9:8.2f} GB", flush=True)
