"""CPU checks of the C-ABI library: it loads, exports every declared symbol,
and its host-side pieces (gate matrices, CRC, FNV) are bit-exact.  No GPU."""
import ctypes as C
import zlib

import numpy as np
import pytest

from conftest import gpu_available
from paper_2309_16979_b200 import engine
from paper_2309_16979_b200.abi import Gate, gate_ptr, to_array


def test_library_loads_and_exports_header_symbols():
    lib = engine.load_library()
    names = engine.exported_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_version_string():
    assert b"sm_100a" in engine.load_library().qzc_version()


def test_gate_matrices_match_reference_golden(golden):
    lib = engine.load_library()
    for rec in golden["matrices"]:
        name, qs, ps = rec["gate"]
        arr = to_array([(name, tuple(qs), tuple(ps))])
        m = np.zeros(16, dtype=np.complex128)
        dim = C.c_uint32()
        assert lib.qzc_gate_matrix(gate_ptr(arr), m.ctypes.data, C.byref(dim)) == 0
        got = m[: dim.value ** 2].view(np.uint64).ravel().tolist()
        assert got == rec["bits"], rec["gate"]


def test_host_crc_and_fnv():
    lib = engine.load_library()
    rng = np.random.default_rng(9)
    for n in (0, 1, 31, 1000):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        p = b.ctypes.data_as(C.POINTER(C.c_uint8))
        assert lib.qzc_crc32(p, n) == zlib.crc32(b.tobytes())
    assert lib.qzc_fnv1a64(None, 0, 0xcbf29ce484222325) == 0xcbf29ce484222325


def test_payload_bound_covers_worst_case():
    lib = engine.load_library()
    # lossless: 8 planes x 2N bytes, one pair (2 B) per byte worst case
    assert lib.qzc_payload_bound(256, 0.0) >= 17 + 8 * 2 * 2 * 256
    assert lib.qzc_payload_bound(256, 1e-5) >= 17 + 2 * 2 * 2 * 256 + 2 * 256 * 8


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_engine_fails_loudly_without_gpu():
    with pytest.raises(engine.QzError):
        engine.Engine()
