"""Wall-clock breakdown of one bench step (init_basis / run) for a circuit."""
import sys
import time

from paper_2309_16979_b200 import circuits
from paper_2309_16979_b200.engine import Engine

circ = sys.argv[1] if len(sys.argv) > 1 else "qft"
fuse = {"strict": "strict", "relaxed": True}[sys.argv[2] if len(sys.argv) > 2 else "relaxed"]
n = 30
eng = Engine()
gates = circuits.make(circ, n)
sim = eng.simulator(n, 16, 30, 1e-5, init=False, fuse=fuse)
for rep in range(4):
    t0 = time.perf_counter()
    sim.init_basis()
    t1 = time.perf_counter()
    sim.run(gates)
    t2 = time.perf_counter()
    st = sim.stats()
    print(f"{circ} {fuse}: init {1e3*(t1-t0):.1f} ms run {1e3*(t2-t1):.1f} ms "
          f"(wall {1e3*st['wall_seconds']:.1f} dec {1e3*st['decode_seconds']:.1f} "
          f"gates {1e3*st['gate_seconds']:.1f} enc {1e3*st['encode_seconds']:.1f}) "
          f"passes {st['gate_passes']} replays {st['replays']}", flush=True)
