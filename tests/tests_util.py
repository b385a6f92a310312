"""Shared helpers for tests (circuits from the golden fixture or seeds)."""
import numpy as np

KINDS = ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "u1", "u2", "u3",
         "cx", "cz", "swap"]
NPAR = {"rx": 1, "ry": 1, "rz": 1, "u1": 1, "u2": 2, "u3": 3}


def random_circuit(n: int, depth: int, seed: int) -> list:
    """Seeded random circuit over the full gate set (numpy PCG64 stream)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(depth):
        k = KINDS[rng.integers(0, len(KINDS))]
        if k in ("cx", "cz", "swap"):
            q = rng.choice(n, 2, replace=False)
            out.append((k, (int(q[0]), int(q[1])), ()))
        else:
            out.append((k, (int(rng.integers(0, n)),),
                        tuple(float(x) for x in rng.uniform(-np.pi, np.pi, NPAR.get(k, 0)))))
    return out
