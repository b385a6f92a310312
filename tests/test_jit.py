"""Runtime-specialised gate passes (qz_jit.cu): the generated source builds
with NVRTC for sm_100a on the host (CPU), and on the GPU the specialised
kernels give the same digests as the AOT kernels (QZ_JIT=0)."""
import ctypes
import os
import subprocess
import sys

import pytest

from paper_2309_16979_b200 import circuits, engine


def _have_nvrtc() -> bool:
    for name in ("libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
        try:
            ctypes.CDLL(name)
            return True
        except OSError:
            pass
    return False


@pytest.mark.skipif(not _have_nvrtc(), reason="libnvrtc not present")
@pytest.mark.parametrize("name", ["qft", "supremacy"])
def test_jit_source_compiles(name):
    gates = circuits.qft(24) if name == "qft" else circuits.supremacy(24, depth=4, seed=3)
    engine.jit_selftest(gates, 24)


_DIGEST = r"""
import json, sys
from paper_2309_16979_b200 import circuits, engine
n = int(sys.argv[1]); which = sys.argv[2]
g = {"qft": lambda: circuits.qft(n), "sup": lambda: circuits.supremacy(n, depth=8, seed=5),
     "grover": lambda: circuits.grover(n)}[which]()
eng = engine.Engine()
out = []
for rnd in range(2):
    sim = engine.Simulator(eng, n, 12, n, 1e-5)
    sim.run(g)
    out.append(sim.digest())
    sim.close()
    engine.jit_wait()
eng.close()
print(json.dumps(out))
"""


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["qft", "sup", "grover"])
def test_jit_matches_aot(which):
    """Same store digest with and without the specialised passes (second run
    in each process uses the kernels the first run queued)."""
    res = {}
    for jit in ("0", "1"):
        env = dict(os.environ, QZ_JIT=jit, QZ_JIT_MIN_BITS="16")
        out = subprocess.run([sys.executable, "-c", _DIGEST, "20", which], env=env, capture_output=True,
                             text=True, timeout=600, check=True)
        res[jit] = out.stdout.strip().splitlines()[-1]
    import json
    a, b = json.loads(res["0"]), json.loads(res["1"])
    assert a[0] == a[1] == b[0] == b[1]
