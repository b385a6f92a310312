"""Run one circuit once through the engine (profiling / debugging helper)."""
import argparse
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from paper_2309_16979_b200 import circuits
from paper_2309_16979_b200.engine import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--circuit", default="qft")
ap.add_argument("--n", type=int, default=28)
ap.add_argument("--c", type=int, default=16)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--eb", type=float, default=1e-5)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
eng = Engine()
g = circuits.make(a.circuit, a.n)
sim = eng.simulator(a.n, a.c, a.m or a.n, a.eb, init=False)
for _ in range(a.reps):
    sim.init_basis()
    t = time.time()
    sim.run(g)
    print(f"{a.circuit}-{a.n}: {time.time() - t:.3f}s", sim.stats(), flush=True)
