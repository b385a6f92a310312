"""Error-bound sweep (cfg5's eb axis; paper Fig. 'ratio / fidelity vs
error bound'): one circuit at n qubits for each error bound, compressed store
HBM-resident, CUDA-event timed; compression ratio, fidelity against an
uncompressed fp64 GPU run of the same circuit (when the dense state fits next
to the store) and gates/s.  One JSON line per error bound.

  python tools/eb_sweep.py --circuit supremacy --n 30 --eb 1e-7 1e-8 1e-9
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import ClockSampler, fidelity_of  # noqa: E402
from paper_2309_16979_b200 import circuits  # noqa: E402
from paper_2309_16979_b200.engine import Engine, jit_wait  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--circuit", default="supremacy")
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--c", type=int, default=16)
ap.add_argument("--m", type=int, default=30)
ap.add_argument("--depth", type=int, default=20)
ap.add_argument("--eb", type=float, nargs="+", default=[1e-7, 1e-8, 1e-9])
ap.add_argument("--reps", type=int, default=2, help="timed runs per error bound (after one warm-up)")
a = ap.parse_args()

eng = Engine()
gates = circuits.supremacy(a.n, depth=a.depth) if a.circuit == "supremacy" else circuits.make(a.circuit, a.n)
for eb in a.eb:
    sim = eng.simulator(a.n, a.c, a.m, eb, init=False)
    sim.init_basis()
    sim.run(gates)          # warm-up (queues the specialised passes)
    jit_wait()
    clk = ClockSampler(0)
    clk.start()
    times = []
    for _ in range(a.reps):
        sim.init_basis()
        eng.timer_begin()
        sim.run(gates)
        times.append(eng.timer_end())
    clocks = clk.stop()
    st = sim.stats()
    out = {"workload": f"{a.circuit}-{a.n}" + (f" depth {a.depth}" if a.circuit == "supremacy" else "") +
                       f" c={a.c} m={a.m}, HBM-resident", "error_bound": eb, "gates": len(gates),
           "seconds": min(times), "gates_per_s": len(gates) / min(times), "stages": st["stages"],
           "compression_ratio": st["ratio"], "store_bytes": sim.payload_bytes(),
           "digest": f"{sim.digest():016x}", "clocks": clocks}
    out.update(fidelity_of(eng, sim, a.n, gates))
    sim.close()
    print(json.dumps(out), flush=True)
