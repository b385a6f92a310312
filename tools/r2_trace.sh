# host-side split of one QFT-30 stage (plan / launch / sync), QZ_TRACE=1
python - <<'PY' 2>&1 | grep -v "pass \|group\|zmask" | tail -30
import os, time
os.environ["QZ_TRACE"] = "1"
from paper_2309_16979_b200 import circuits
from paper_2309_16979_b200.engine import Engine, jit_wait
eng = Engine()
g = circuits.make("qft", 30)
sim = eng.simulator(30, 16, 30, 1e-5, init=False)
for rep in range(4):
    sim.init_basis()
    t0 = time.perf_counter()
    sim.run(g)
    print("run wall %.2f ms" % (1e3 * (time.perf_counter() - t0)), flush=True)
    if rep == 0:
        jit_wait()
PY
