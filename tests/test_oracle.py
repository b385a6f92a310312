"""The CPU oracle (oracle/qz_oracle.c) against the reference's golden vectors.

The fixture (tests/golden/golden.json) was produced by the unmodified
reference through oracle/_ref (tests/golden/make_golden.py).  These tests pin
the restatement before it is trusted as the GPU checker.
"""
import hashlib

import numpy as np
import pytest

from golden.inputs import CODEC_CASES, KERNEL_CASES, codec_input, kernel_input
from paper_2309_16979_b200.abi import to_array


def circ(golden, key):
    return to_array([(g[0], tuple(g[1]), tuple(g[2])) for g in golden["circuits"][key]])


def test_fixture_covers_inputs(golden):
    assert len(golden["codec"]) == len(CODEC_CASES)
    assert len(golden["kernels"]) == len(KERNEL_CASES)


def test_matrices_bitwise(golden, oracle):
    for rec in golden["matrices"]:
        name, qs, ps = rec["gate"]
        m = oracle.gate_matrix((name, tuple(qs), tuple(ps)))
        assert m.view(np.uint64).ravel().tolist() == rec["bits"], rec["gate"]


def test_reference_known_answer_ones(oracle):
    # test_codec.cpp:74-98 — reals [1,1,1,1] at eb=0.1
    payload, _ = oracle.compress(np.ones(4, complex), 0.1)
    expect = bytes([1]) + np.float64(0.1).tobytes() + bytes([4, 0, 0, 0, 0, 0, 0, 0]) + \
        bytes([10, 1, 0, 7, 0, 8])
    assert payload == expect


def test_reference_known_answer_zero_chunk(oracle):
    # test_codec.cpp:186-193 — zero c=16 chunk is 2077 bytes
    payload, _ = oracle.compress(np.zeros(1 << 16, complex), 1e-5)
    assert len(payload) == 2077


@pytest.mark.parametrize("idx", range(len(CODEC_CASES)))
def test_codec_golden(golden, oracle, idx):
    case = CODEC_CASES[idx]
    rec = golden["codec"][idx]
    amps, forced = codec_input(case)
    payload, crc = oracle.compress(amps, case["eb"], forced)
    assert len(payload) == rec["len"]
    assert crc == rec["crc"]
    assert hashlib.sha256(payload).hexdigest() == rec["sha256"]
    back = oracle.decompress(payload, crc, amps.size)
    assert hashlib.sha256(back.tobytes()).hexdigest() == rec["decoded_sha256"]


@pytest.mark.parametrize("idx", range(len(KERNEL_CASES)))
def test_kernels_golden(golden, oracle, idx):
    rec = golden["kernels"][idx]
    buf = kernel_input(KERNEL_CASES[idx])
    gates = to_array([(g[0], tuple(g[1]), tuple(g[2])) for g in rec["gates"]])
    out = oracle.apply_gates(buf, gates)
    assert hashlib.sha256(out.tobytes()).hexdigest() == rec["sha256"]


def test_runs_small_golden(golden, oracle):
    for rec in golden["runs_small"]:
        r = oracle.run(rec["n"], circ(golden, rec["circuit"]), rec["c"], rec["m"], rec["eb"])
        assert f"{r['digest']:016x}" == rec["digest"], rec
        assert r["stages"] == rec["stages"]
        assert r["current_bytes"] == rec["current_bytes"]
        assert r["peak_bytes"] == rec["peak_bytes"]
        assert r["norm"] == pytest.approx(rec["norm"], abs=1e-12)


def test_runs_golden(golden, oracle):
    for rec in golden["runs"]:
        if rec["n"] > 20:
            continue  # the single-threaded oracle is slow beyond 20 qubits
        key = rec["circuit"]
        if key.startswith("qft:"):
            g = oracle.make_qft(int(key.split(":")[1]))
        elif key.startswith("ghz:"):
            g = oracle.make_ghz(int(key.split(":")[1]))
        else:
            g = circ(golden, key)
        r = oracle.run(rec["n"], g, rec["c"], rec["m"], rec["eb"])
        assert f"{r['digest']:016x}" == rec["digest"], rec
        assert r["stages"] == rec["stages"]
        assert r["total_payload"] == rec["total_payload"]


def test_generators(golden, oracle):
    for n, gl in golden["generators"]["qft"].items():
        assert oracle.make_qft(int(n)).tobytes() == circ_list(gl).tobytes()
    for n, gl in golden["generators"]["ghz"].items():
        assert oracle.make_ghz(int(n)).tobytes() == circ_list(gl).tobytes()


def circ_list(gl):
    return to_array([(g[0], tuple(g[1]), tuple(g[2])) for g in gl])


def test_crc_and_fnv(oracle):
    import zlib
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 100, 4099):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert oracle.crc32(b) == zlib.crc32(b)
    assert oracle.fnv1a64(b"") == 0xcbf29ce484222325
    assert oracle.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
