"""Benchmark circuit families (inputs to the hot path, emitted in the
reference's gate set, include/qzsim/gates.hpp:27-45).

* ``qft`` / ``ghz`` restate generators.cpp:21-59 gate for gate (the QFT's
  controlled phases decomposed into U1/CX exactly as push_controlled_phase,
  generators.cpp:32-40), so the same circuits reach the reference and the
  engine and the golden digests apply.
* ``supremacy`` / ``qaoa`` / ``grover`` are the new families BASELINE.json's
  configs 3-4 name; they use only reference gates (no CCX: SPEC.md:68).
* ``to_qasm`` emits OpenQASM 2.0 text with %.17g angles, the format
  qzsim's parser and pretty_print round-trip exactly (qasm.cpp:304-308).
"""
from __future__ import annotations

import math

import numpy as np

from .abi import to_array


def ghz(n: int) -> np.ndarray:
    gates = [("h", (0,), ())] + [("cx", (0, k), ()) for k in range(1, n)]
    return to_array(gates)


def _controlled_phase(out: list, lam: float, a: int, b: int) -> None:
    out.append(("u1", (a,), (lam / 2.0,)))
    out.append(("cx", (a, b), ()))
    out.append(("u1", (b,), (-lam / 2.0,)))
    out.append(("cx", (a, b), ()))
    out.append(("u1", (b,), (lam / 2.0,)))


def qft(n: int) -> np.ndarray:
    out: list = []
    for i in range(n):
        target = n - 1 - i
        out.append(("h", (target,), ()))
        for j in range(target):
            control = target - 1 - j
            _controlled_phase(out, math.pi / float(1 << (j + 1)), control, target)
    for i in range(n // 2):
        out.append(("swap", (i, n - 1 - i), ()))
    return to_array(out)


def supremacy(n: int, depth: int = 20, seed: int = 1) -> np.ndarray:
    """Supremacy-style layers: a random single-qubit gate from
    {RX(pi/2), RY(pi/2), U2(0, pi/4)-type} on every qubit, then CZ on
    alternating nearest-neighbour pairs (brick pattern)."""
    rng = np.random.default_rng(seed)
    singles = [("rx", (math.pi / 2,)), ("ry", (math.pi / 2,)), ("u2", (0.0, math.pi / 4))]
    out: list = []
    for layer in range(depth):
        for q in range(n):
            name, ps = singles[int(rng.integers(0, 3))]
            out.append((name, (q,), ps))
        for q in range(layer % 2, n - 1, 2):
            out.append(("cz", (q, q + 1), ()))
    return to_array(out)


def qaoa(n: int, p: int = 2, seed: int = 1) -> np.ndarray:
    """QAOA MaxCut on a random 3-regular-ish graph: H layer, then p rounds of
    RZZ(gamma) via CX-RZ-CX per edge and RX(2 beta) mixers."""
    rng = np.random.default_rng(seed)
    edges = set()
    for q in range(n):
        for _ in range(2):
            r = int(rng.integers(0, n))
            if r != q:
                edges.add((min(q, r), max(q, r)))
    edges = sorted(edges)
    out: list = [("h", (q,), ()) for q in range(n)]
    for _ in range(p):
        gamma, beta = float(rng.uniform(0, math.pi)), float(rng.uniform(0, math.pi))
        for a, b in edges:
            out += [("cx", (a, b), ()), ("rz", (b,), (gamma,)), ("cx", (a, b), ())]
        out += [("rx", (q,), (2 * beta,)) for q in range(n)]
    return to_array(out)


def _ccx(out: list, a: int, b: int, c: int) -> None:
    """Toffoli in {H, T, TDG, CX} (the standard exact 7-T decomposition)."""
    out += [("h", (c,), ()), ("cx", (b, c), ()), ("tdg", (c,), ()), ("cx", (a, c), ()),
            ("t", (c,), ()), ("cx", (b, c), ()), ("tdg", (c,), ()), ("cx", (a, c), ()),
            ("t", (b,), ()), ("t", (c,), ()), ("h", (c,), ()), ("cx", (a, b), ()),
            ("t", (a,), ()), ("tdg", (b,), ()), ("cx", (a, b), ())]


def _mcx(out: list, controls: list, target: int, ancillas: list) -> None:
    """Multi-controlled X by a V-chain of Toffolis over len(controls)-2 clean
    ancillas, uncomputed afterwards."""
    k = len(controls)
    if k == 1:
        out.append(("cx", (controls[0], target), ()))
        return
    if k == 2:
        _ccx(out, controls[0], controls[1], target)
        return
    chain = []
    _ccx(out, controls[0], controls[1], ancillas[0])
    chain.append((controls[0], controls[1], ancillas[0]))
    for i in range(2, k - 1):
        _ccx(out, controls[i], ancillas[i - 2], ancillas[i - 1])
        chain.append((controls[i], ancillas[i - 2], ancillas[i - 1]))
    _ccx(out, controls[k - 1], ancillas[k - 3], target)
    for a, b, c in reversed(chain):
        _ccx(out, a, b, c)


def grover(n: int, iterations: int = 1, marked: int = 0) -> np.ndarray:
    """Grover search over an r-qubit register with r-3 clean ancillas
    (2r - 3 <= n): phase oracle on |marked>, then the diffusion operator.
    The multi-controlled Z is H · MCX · H with the MCX built from exact
    Toffolis (no CCX kind in the reference gate set)."""
    r = max(2, (n + 3) // 2)
    reg = list(range(r))
    anc = list(range(r, n))
    assert len(anc) >= max(0, r - 3), "not enough qubits for the ancilla chain"
    out: list = [("h", (q,), ()) for q in reg]

    def mcz() -> None:
        out.append(("h", (reg[-1],), ()))
        _mcx(out, reg[:-1], reg[-1], anc)
        out.append(("h", (reg[-1],), ()))

    for _ in range(iterations):
        out.extend(("x", (q,), ()) for q in reg if not (marked >> q) & 1)
        mcz()
        out.extend(("x", (q,), ()) for q in reg if not (marked >> q) & 1)
        out.extend(("h", (q,), ()) for q in reg)
        out.extend(("x", (q,), ()) for q in reg)
        mcz()
        out.extend(("x", (q,), ()) for q in reg)
        out.extend(("h", (q,), ()) for q in reg)
    return to_array(out)


FAMILIES = {"qft": qft, "ghz": ghz, "supremacy": supremacy, "qaoa": qaoa, "grover": grover}


def make(family: str, n: int, **kw) -> np.ndarray:
    return FAMILIES[family](n, **kw)


def to_qasm(n: int, gates, reg: str = "q") -> str:
    from .abi import from_array
    lines = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg {reg}[{n}];"]
    for name, qs, ps in from_array(to_array(gates)):
        args = ",".join(f"{reg}[{q}]" for q in qs)
        par = "(" + ",".join("%.17g" % p for p in ps) + ")" if ps else ""
        lines.append(f"{name}{par} {args};")
    return "\n".join(lines) + "\n"
