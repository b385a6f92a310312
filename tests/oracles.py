"""Test-side bindings to the two CPU checkers (never imported by the product).

* ``Oracle``    — oracle/liboracle.so, the C restatement (oracle/qz_oracle.c).
* ``Reference`` — oracle/_ref/libqzref.so, the UNMODIFIED reference sources
  compiled by oracle/Makefile (only present where it was built; it travels to
  the GPU box as a built artefact).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import sys

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_16979_b200.abi import Gate, gate_ptr, to_array

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libqzref.so"

P = C.POINTER
u8p, u32p, u64p, f64p = P(C.c_uint8), P(C.c_uint32), P(C.c_uint64), P(C.c_double)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _amps(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a


class CodecFailure(Exception):
    pass


class Oracle:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        lib = C.CDLL(str(path))
        lib.qzo_compress.restype = C.c_int64
        lib.qzo_compress.argtypes = [C.c_void_p, C.c_uint64, C.c_double, u64p,
                                     C.c_uint64, u8p, C.c_uint64, u32p]
        lib.qzo_decompress.restype = C.c_int
        lib.qzo_decompress.argtypes = [u8p, C.c_uint64, C.c_uint32, C.c_uint64,
                                       C.c_void_p, C.c_char_p, C.c_size_t]
        lib.qzo_payload_bound.restype = C.c_uint64
        lib.qzo_payload_bound.argtypes = [C.c_uint64]
        lib.qzo_crc32.restype = C.c_uint32
        lib.qzo_crc32.argtypes = [u8p, C.c_size_t]
        lib.qzo_fnv1a64.restype = C.c_uint64
        lib.qzo_fnv1a64.argtypes = [u8p, C.c_size_t, C.c_uint64]
        lib.qzo_gate_matrix.argtypes = [P(Gate), C.c_void_p, u32p]
        lib.qzo_apply_gates.argtypes = [C.c_void_p, C.c_uint64, P(Gate), C.c_uint64]
        lib.qzo_make_qft.restype = C.c_uint64
        lib.qzo_make_qft.argtypes = [C.c_uint32, P(Gate), C.c_uint64]
        lib.qzo_make_ghz.restype = C.c_uint64
        lib.qzo_make_ghz.argtypes = [C.c_uint32, P(Gate), C.c_uint64]
        lib.qzo_run.argtypes = [C.c_uint32, P(Gate), C.c_uint64, C.c_uint32, C.c_uint32,
                                C.c_double, C.c_void_p, u8p, C.c_uint64, u32p]
        lib.qzo_dense.argtypes = [C.c_uint32, P(Gate), C.c_uint64, C.c_void_p]
        lib.qzo_fidelity.restype = C.c_double
        lib.qzo_fidelity.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        self.lib = lib

    # codec.cpp:95-185
    def compress(self, amps, eb: float, forced=()) -> tuple[bytes, int]:
        a = _amps(amps)
        n = a.size
        forced = np.ascontiguousarray(np.asarray(forced, dtype=np.uint64))
        cap = int(self.lib.qzo_payload_bound(max(n, 1)))
        out = np.zeros(cap, dtype=np.uint8)
        crc = C.c_uint32()
        r = self.lib.qzo_compress(a.ctypes.data, n, eb, _ptr(forced, u64p), forced.size,
                                  _ptr(out, u8p), cap, C.byref(crc))
        if r < 0:
            raise CodecFailure(f"compress failed {r}")
        return out[:r].tobytes(), crc.value

    def decompress(self, payload: bytes, crc: int, n: int) -> np.ndarray:
        p = np.frombuffer(payload, dtype=np.uint8).copy()
        out = np.zeros(n, dtype=np.complex128)
        err = C.create_string_buffer(256)
        r = self.lib.qzo_decompress(_ptr(p, u8p), p.size, crc, n, out.ctypes.data, err, 256)
        if r:
            raise CodecFailure(err.value.decode())
        return out

    def crc32(self, b: bytes) -> int:
        p = np.frombuffer(b, dtype=np.uint8).copy()
        return self.lib.qzo_crc32(_ptr(p, u8p), p.size)

    def fnv1a64(self, b: bytes, state: int = 0xcbf29ce484222325) -> int:
        p = np.frombuffer(b, dtype=np.uint8).copy()
        return self.lib.qzo_fnv1a64(_ptr(p, u8p), p.size, state)

    def gate_matrix(self, g) -> np.ndarray:
        arr = to_array([g])
        m = np.zeros(16, dtype=np.complex128)
        dim = C.c_uint32()
        assert self.lib.qzo_gate_matrix(gate_ptr(arr), m.ctypes.data, C.byref(dim)) == 0
        return m[: dim.value * dim.value].reshape(dim.value, dim.value)

    def apply_gates(self, amps, gates) -> np.ndarray:
        a = _amps(amps).copy()
        arr = to_array(gates)
        assert self.lib.qzo_apply_gates(a.ctypes.data, a.size, gate_ptr(arr), arr.size) == 0
        return a

    def make_qft(self, n: int) -> np.ndarray:
        cnt = self.lib.qzo_make_qft(n, None, 0)
        arr = np.zeros(cnt, dtype=to_array([]).dtype)
        self.lib.qzo_make_qft(n, gate_ptr(arr), cnt)
        return arr

    def make_ghz(self, n: int) -> np.ndarray:
        cnt = self.lib.qzo_make_ghz(n, None, 0)
        arr = np.zeros(cnt, dtype=to_array([]).dtype)
        self.lib.qzo_make_ghz(n, gate_ptr(arr), cnt)
        return arr

    def run(self, n, gates, c, m, eb, export=False) -> dict:
        arr = to_array(gates)
        res = (C.c_uint64 * 8)()
        nchunks = 1 << (n - c)
        sizes = np.zeros(nchunks, dtype=np.uint32)
        cap = int(self.lib.qzo_payload_bound(1 << c)) * nchunks if export else 0
        out = np.zeros(max(cap, 1), dtype=np.uint8)
        r = self.lib.qzo_run(n, gate_ptr(arr), arr.size, c, m, eb, C.addressof(res),
                             _ptr(out, u8p) if export else None, cap, _ptr(sizes, u32p))
        if r:
            raise RuntimeError(f"oracle run failed {r}")
        raw = bytes(res)
        digest, _, cur, peak, dense, stages, total = np.frombuffer(raw[:56], dtype=np.uint64)
        norm = np.frombuffer(raw[8:16], dtype=np.float64)[0]
        secs = np.frombuffer(raw[56:64], dtype=np.float64)[0]
        d = dict(digest=int(digest), norm=float(norm), current_bytes=int(cur),
                 peak_bytes=int(peak), dense_bytes=int(dense), stages=int(stages),
                 total_payload=int(total), seconds=float(secs), sizes=sizes)
        if export:
            d["payload"] = out[: int(total)].tobytes()
        return d

    def dense(self, n, gates) -> np.ndarray:
        arr = to_array(gates)
        out = np.zeros(1 << n, dtype=np.complex128)
        assert self.lib.qzo_dense(n, gate_ptr(arr), arr.size, out.ctypes.data) == 0
        return out

    def fidelity(self, a, b) -> float:
        a, b = _amps(a), _amps(b)
        return self.lib.qzo_fidelity(a.ctypes.data, b.ctypes.data, a.size)


class RefResult(C.Structure):
    _fields_ = [("digest", C.c_uint64), ("norm", C.c_double), ("wall_seconds", C.c_double),
                ("ratio", C.c_double), ("current_bytes", C.c_uint64),
                ("peak_bytes", C.c_uint64), ("stages", C.c_uint64),
                ("total_payload", C.c_uint64), ("fidelity", C.c_double)]


class Reference:
    """The reference library itself (oracle/_ref/libqzref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        lib = C.CDLL(str(path))
        lib.qzref_last_error.restype = C.c_char_p
        lib.qzref_compress.restype = C.c_int64
        lib.qzref_compress.argtypes = [C.c_void_p, C.c_uint64, C.c_double, u64p,
                                       C.c_uint64, u8p, C.c_uint64, u32p]
        lib.qzref_decompress.argtypes = [u8p, C.c_uint64, C.c_uint32, C.c_uint64,
                                         C.c_uint64, C.c_void_p]
        lib.qzref_gate_matrix.argtypes = [P(Gate), C.c_void_p, u32p]
        lib.qzref_apply_gates.argtypes = [C.c_void_p, C.c_uint64, P(Gate), C.c_uint64]
        for f in ("qzref_make_qft", "qzref_make_ghz"):
            getattr(lib, f).restype = C.c_uint64
            getattr(lib, f).argtypes = [C.c_uint32, P(Gate), C.c_uint64]
        lib.qzref_make_random.restype = C.c_uint64
        lib.qzref_make_random.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, P(Gate),
                                          C.c_uint64]
        lib.qzref_plan.argtypes = [C.c_uint32, P(Gate), C.c_uint64, C.c_uint32, C.c_uint32,
                                   u64p, u64p, u32p, u32p, C.c_uint64]
        lib.qzref_run.argtypes = [C.c_uint32, P(Gate), C.c_uint64, C.c_uint32, C.c_uint32,
                                  C.c_double, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.c_uint32, P(RefResult), u8p, C.c_uint64, u32p]
        self.lib = lib

    def err(self) -> str:
        return self.lib.qzref_last_error().decode()

    def compress(self, amps, eb: float, forced=()) -> tuple[bytes, int]:
        a = _amps(amps)
        forced = np.ascontiguousarray(np.asarray(forced, dtype=np.uint64))
        cap = 40 * max(a.size, 1) + 64
        out = np.zeros(cap, dtype=np.uint8)
        crc = C.c_uint32()
        r = self.lib.qzref_compress(a.ctypes.data, a.size, eb, _ptr(forced, u64p),
                                    forced.size, _ptr(out, u8p), cap, C.byref(crc))
        if r < 0:
            raise CodecFailure(self.err())
        return out[:r].tobytes(), crc.value

    def decompress(self, payload: bytes, crc: int, n: int, chunk_index: int = 0) -> np.ndarray:
        p = np.frombuffer(payload, dtype=np.uint8).copy()
        out = np.zeros(n, dtype=np.complex128)
        if self.lib.qzref_decompress(_ptr(p, u8p), p.size, crc, n, chunk_index,
                                     out.ctypes.data):
            raise CodecFailure(self.err())
        return out

    def gate_matrix(self, g) -> np.ndarray:
        arr = to_array([g])
        m = np.zeros(16, dtype=np.complex128)
        dim = C.c_uint32()
        assert self.lib.qzref_gate_matrix(gate_ptr(arr), m.ctypes.data, C.byref(dim)) == 0
        return m[: dim.value * dim.value].reshape(dim.value, dim.value)

    def apply_gates(self, amps, gates) -> np.ndarray:
        a = _amps(amps).copy()
        arr = to_array(gates)
        assert self.lib.qzref_apply_gates(a.ctypes.data, a.size, gate_ptr(arr), arr.size) == 0
        return a

    def _gen(self, f, *args) -> np.ndarray:
        cnt = f(*args, None, 0)
        arr = np.zeros(cnt, dtype=to_array([]).dtype)
        f(*args, gate_ptr(arr), cnt)
        return arr

    def make_qft(self, n): return self._gen(self.lib.qzref_make_qft, n)
    def make_ghz(self, n): return self._gen(self.lib.qzref_make_ghz, n)
    def make_random(self, n, depth, seed): return self._gen(self.lib.qzref_make_random, n, depth, seed)

    def plan(self, n, gates, c, m):
        arr = to_array(gates)
        cap = max(arr.size, 1)
        ns = C.c_uint64()
        sng = np.zeros(cap, dtype=np.uint64)
        nh = np.zeros(cap, dtype=np.uint32)
        hi = np.zeros(cap * 64, dtype=np.uint32)
        if self.lib.qzref_plan(n, gate_ptr(arr), arr.size, c, m, C.byref(ns), _ptr(sng, u64p),
                               _ptr(nh, u32p), _ptr(hi, u32p), cap):
            raise ValueError(self.err())
        return [(int(sng[s]), [int(x) for x in hi[s * 64: s * 64 + nh[s]]])
                for s in range(ns.value)]

    def run(self, n, gates, c, m, eb, workers=0, depth=2, strategy=2, oracle_limit=0,
            export=False) -> dict:
        arr = to_array(gates)
        res = RefResult()
        nchunks = 1 << (n - c)
        sizes = np.zeros(nchunks, dtype=np.uint32)
        cap = (40 * (1 << c) + 64) * nchunks if export else 0
        out = np.zeros(max(cap, 1), dtype=np.uint8)
        r = self.lib.qzref_run(n, gate_ptr(arr), arr.size, c, m, eb, workers, depth, strategy,
                               oracle_limit, C.byref(res), _ptr(out, u8p) if export else None,
                               cap, _ptr(sizes, u32p))
        if r:
            raise RuntimeError(self.err())
        d = {name: getattr(res, name) for name, _ in RefResult._fields_}
        d["sizes"] = sizes
        if export:
            d["payload"] = out[: res.total_payload].tobytes()
        return d


def have_reference() -> bool:
    return REF_SO.exists()
