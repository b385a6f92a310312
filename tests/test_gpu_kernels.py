"""GPU gate kernels: bit-identical to the reference's apply_gates
(kernels.cpp:20-68) on the golden buffers, fused and per-gate passes.
Mirrors test_device.cpp:119-204."""
import hashlib

import numpy as np
import pytest

from golden.inputs import KERNEL_CASES, kernel_input
from paper_2309_16979_b200 import engine as E
from paper_2309_16979_b200.abi import to_array

pytestmark = pytest.mark.gpu


def gl(rec):
    return to_array([(g[0], tuple(g[1]), tuple(g[2])) for g in rec])


def test_golden_kernel_cases(engine, golden):
    for case, rec in zip(KERNEL_CASES, golden["kernels"]):
        buf = kernel_input(case)
        out = engine.apply_gates(buf, gl(rec["gates"]))
        assert hashlib.sha256(out.tobytes()).hexdigest() == rec["sha256"], case


@pytest.mark.parametrize("nbits", [2, 5, 9, 13, 16, 20])
def test_random_circuits_vs_oracle(engine, oracle, golden, nbits):
    rng = np.random.default_rng(nbits)
    kinds = ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "u1", "u2", "u3",
             "cx", "cz", "swap"]
    gates = []
    for _ in range(150):
        k = kinds[rng.integers(0, len(kinds))]
        if k in ("cx", "cz", "swap"):
            q = rng.choice(nbits, 2, replace=False)
            gates.append((k, (int(q[0]), int(q[1])), ()))
        else:
            npar = {"rx": 1, "ry": 1, "rz": 1, "u1": 1, "u2": 2, "u3": 3}.get(k, 0)
            gates.append((k, (int(rng.integers(0, nbits)),), tuple(rng.uniform(-4, 4, npar))))
    a = rng.uniform(-1, 1, 1 << nbits) + 1j * rng.uniform(-1, 1, 1 << nbits)
    a[rng.integers(0, 1 << nbits, 1 << max(0, nbits - 3))] = 0.0   # exact zeros: ±0 rules
    a[::5] = -0.0
    ref = oracle.apply_gates(a, gates)
    got = engine.apply_gates(a, gates)
    assert got.tobytes() == ref.tobytes()


def test_h_and_cx_truth(engine):
    out = engine.apply_gates(np.array([1, 0], complex), [("h", (0,), ())])
    r = 1 / np.sqrt(2)
    assert abs(out[0] - r) <= 1e-15 and abs(out[1] - r) <= 1e-15
    buf = np.array([0, 0, 1, 0], complex)  # |10>, CX(control 1, target 0) -> |11>
    out = engine.apply_gates(buf, [("cx", (1, 0), ())])
    assert out[2] == 0 and out[3] == 1


def test_ghz_basis_zero_signs(engine, oracle):
    # basis / GHZ states are mostly exact zeros: zero signs must match
    n = 12
    a = np.zeros(1 << n, complex)
    a[0] = 1
    g = oracle.make_ghz(n)
    assert engine.apply_gates(a, g).tobytes() == oracle.apply_gates(a, g).tobytes()
    q = oracle.make_qft(n)
    assert engine.apply_gates(a, q).tobytes() == oracle.apply_gates(a, q).tobytes()


def test_linearity(engine):
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, 256) + 1j * rng.uniform(-1, 1, 256)
    y = rng.uniform(-1, 1, 256) + 1j * rng.uniform(-1, 1, 256)
    al, be = 0.3 - 0.2j, -1.1 + 0.7j
    g = [("u3", (3,), (0.3, 1.0, -0.5)), ("cx", (2, 7), ()), ("rx", (0,), (1.1,))]
    fx, fy = engine.apply_gates(x, g), engine.apply_gates(y, g)
    fc = engine.apply_gates(al * x + be * y, g)
    assert np.abs(fc - (al * fx + be * fy)).max() <= 1e-12


def test_bad_bit_fails(engine):
    with pytest.raises(E.DeviceError):
        engine.apply_gates(np.zeros(16, complex), [("h", (4,), ())])


@pytest.mark.parametrize("nbits,dim", [(10, 2), (14, 2), (12, 4), (15, 4)])
def test_sub_range_apply_matches_whole_gate(engine, oracle, nbits, dim):
    """apply_single_qubit / apply_two_qubit sub-ranges (kernels.cpp:20-54,
    the reference's worker split) through qzc_apply_matrix_range_host: the
    union of the ranges equals the whole gate bit for bit (the reference's
    apply_gates, via the C oracle), and amplitudes outside a range stay
    untouched."""
    import ctypes as C
    from paper_2309_16979_b200.abi import to_array
    lib = engine.lib
    lib.qzc_apply_matrix_range_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                                C.c_uint64, C.c_uint64]
    rng = np.random.default_rng(nbits * dim)
    buf = (rng.standard_normal(1 << nbits) + 1j * rng.standard_normal(1 << nbits)) / 7.0
    buf[rng.integers(0, buf.size, 40)] = 0.0
    for trial in range(6):
        if dim == 2:
            q = (int(rng.integers(0, nbits)),)
            g = ("u3", q, tuple(rng.uniform(-3, 3, 3)))
        else:
            q = tuple(int(x) for x in rng.choice(nbits, 2, replace=False))
            g = (["cx", "cz", "swap"][trial % 3], q, ())
        mat = engine.gate_matrix(g)

        class MG(C.Structure):
            _fields_ = [("dim", C.c_uint32), ("qubits", C.c_uint32 * 2), ("reserved", C.c_uint32),
                        ("m", C.c_double * 32)]
        mg = MG(dim=dim)
        mg.qubits[0] = q[0]
        mg.qubits[1] = q[1] if dim == 4 else 0
        for e, v in enumerate(mat.ravel()):
            mg.m[2 * e], mg.m[2 * e + 1] = v.real, v.imag
        units = (1 << nbits) // dim
        cuts = sorted({0, units, *(int(x) for x in rng.integers(0, units, 3))})
        got = buf.copy()
        for a, b in zip(cuts[:-1], cuts[1:]):
            assert lib.qzc_apply_matrix_range_host(engine.h, got.ctypes.data, nbits, C.byref(mg), a, b) == 0
        want = oracle.apply_gates(buf, to_array([g]))
        assert got.tobytes() == want.tobytes(), (g, cuts)
        # a partial range leaves the other units' amplitudes alone
        part = buf.copy()
        assert lib.qzc_apply_matrix_range_host(engine.h, part.ctypes.data, nbits, C.byref(mg), 0,
                                               units // 2) == 0
        assert (part != buf).any() or g[0] == "cz"
        buf = want
