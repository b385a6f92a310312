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


def diagonal_heavy_circuit(n: int, depth: int, seed: int) -> list:
    """Seeded circuit rich in diagonal units (1q phases, CZ, the CP5 and CXD
    runs the gate passes fold) mixed with H / X / RX so zeros and -0 appear
    and disappear: exercises relaxed passes and their strict replay."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(depth):
        r = int(rng.integers(0, 10))
        a, b = (int(x) for x in rng.choice(n, 2, replace=False))
        lam = float(rng.uniform(-np.pi, np.pi))
        if r == 0:
            out.append(("h", (a,), ()))
        elif r == 1:
            out.append(("x", (a,), ()) if rng.integers(0, 2) else ("rx", (a,), (lam,)))
        elif r == 2:
            out.append((["z", "s", "sdg", "t", "tdg"][int(rng.integers(0, 5))], (a,), ()))
        elif r == 3:
            out.append((["rz", "u1"][int(rng.integers(0, 2))], (a,), (lam,)))
        elif r == 4:
            out.append(("cz", (a, b), ()))
        elif r in (5, 6):
            out += [("u1", (a,), (lam / 2,)), ("cx", (a, b), ()), ("u1", (b,), (-lam / 2,)),
                    ("cx", (a, b), ()), ("u1", (b,), (lam / 2,))]
        elif r == 7:
            out += [("cx", (a, b), ()), ("rz", (b,), (lam,)), ("cx", (a, b), ())]
        elif r == 8:
            out += [("cx", (a, b), ()), ("z", (b,), ()), ("cx", (a, b), ())]
        else:
            out.append(("ry", (a,), (lam,)))
    return out
