"""Wall-clock of the end-to-end step pieces: init + run + export."""
import ctypes as C
import time

import numpy as np

from paper_2309_16979_b200 import circuits
from paper_2309_16979_b200.engine import Engine, u8p, u32p, _check

eng = Engine()
gates = circuits.make("qft", 30)
sim = eng.simulator(30, 16, 30, 1e-5, init=False)
for rep in range(3):
    t0 = time.perf_counter()
    sim.init_basis()
    sim.run(gates)
    t1 = time.perf_counter()
    total = sim.payload_bytes()
    t2 = time.perf_counter()
    buf = np.empty(total, np.uint8)
    sizes = np.empty(sim.chunk_count, np.uint32)
    crcs = np.empty(sim.chunk_count, np.uint32)
    t3 = time.perf_counter()
    _check(sim.lib.qzc_sim_export(sim.h, buf.ctypes.data_as(u8p), buf.size,
                                  sizes.ctypes.data_as(u32p), crcs.ctypes.data_as(u32p)))
    t4 = time.perf_counter()
    b = buf.tobytes()
    t5 = time.perf_counter()
    _check(sim.lib.qzc_sim_export(sim.h, buf.ctypes.data_as(u8p), buf.size,
                                  sizes.ctypes.data_as(u32p), crcs.ctypes.data_as(u32p)))
    t6 = time.perf_counter()
    print(f"init+run {1e3*(t1-t0):.1f} payload_bytes {1e3*(t2-t1):.2f} alloc {1e3*(t3-t2):.2f} "
          f"export {1e3*(t4-t3):.2f} tobytes {1e3*(t5-t4):.2f} export-again {1e3*(t6-t5):.2f} ms", flush=True)
