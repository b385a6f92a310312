"""Multi-stage HBM-resident run (dense decode / encode every stage)."""
import sys
import time

from paper_2309_16979_b200 import circuits
from paper_2309_16979_b200.engine import Engine

circ, n, m, depth = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
eng = Engine()
gates = circuits.supremacy(n, depth=depth) if circ == "supremacy" else circuits.make(circ, n)
sim = eng.simulator(n, 16, m, 1e-7, init=False)
for rep in range(2):
    t0 = time.perf_counter()
    sim.init_basis()
    sim.run(gates)
    st = sim.stats()
    print(f"{circ}-{n} m={m}: {1e3*(time.perf_counter()-t0):.1f} ms stages {st['stages']} windows {st['windows']} "
          f"dec {st['decode_seconds']:.3f} gates {st['gate_seconds']:.3f} enc {st['encode_seconds']:.3f}", flush=True)
