"""Python binding of the sm_100a engine (lib/libqzcuda.so, include/qzcuda.h).

The product path: every call here goes through the C ABI into CUDA kernels.
There is no CPU fallback — if the shared library or a GPU is missing, calls
raise.  Error classes mirror the reference's exception hierarchy
(include/qzsim/util.hpp:34-37 and the per-module *Error types).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .abi import GATE_DTYPE, Gate, KProfRecord, SimConfig, SimStats, gate_ptr, to_array

# QZC_LIB: an alternative build of the same library (tuning experiments)
LIB_PATH = Path(os.environ.get("QZC_LIB", Path(__file__).resolve().parent / "lib" / "libqzcuda.so"))

P = C.POINTER
u8p, u32p, u64p, f64p = P(C.c_uint8), P(C.c_uint32), P(C.c_uint64), P(C.c_double)


class QzError(RuntimeError):
    """Base error (reference: qzsim::Error)."""


class CodecError(QzError):
    pass


class StoreError(QzError):
    pass


class PlanError(QzError):
    pass


class DeviceError(QzError):
    pass


class CudaError(QzError):
    pass


class ArenaFull(QzError):
    pass


_ERRORS = {-1: QzError, -2: CodecError, -3: StoreError, -4: PlanError, -5: DeviceError,
           -6: CudaError, -7: ArenaFull}

_lib = None


def load_library() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build())")
    lib = C.CDLL(str(LIB_PATH))
    sig = {
        "qzc_last_error": (C.c_char_p, []),
        "qzc_version": (C.c_char_p, []),
        "qzc_gate_matrix": (C.c_int, [P(Gate), C.c_void_p, u32p]),
        "qzc_context_create": (C.c_int, [C.c_int, C.c_uint64, P(C.c_void_p)]),
        "qzc_context_destroy": (None, [C.c_void_p]),
        "qzc_synchronize": (C.c_int, [C.c_void_p]),
        "qzc_kernel_launches": (C.c_uint64, [C.c_void_p]),
        "qzc_payload_bound": (C.c_uint64, [C.c_uint64, C.c_double]),
        "qzc_timer_begin": (C.c_int, [C.c_void_p]),
        "qzc_timer_end": (C.c_int, [C.c_void_p, f64p]),
        "qzc_compress_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                        C.c_double, u64p, C.c_uint64, u8p, C.c_uint64, u64p,
                                        u32p, u32p]),
        "qzc_decompress_host": (C.c_int, [C.c_void_p, u8p, u64p, u32p, u32p, C.c_uint64,
                                          C.c_uint64, C.c_uint64, C.c_void_p]),
        "qzc_crc32": (C.c_uint32, [u8p, C.c_uint64]),
        "qzc_fnv1a64": (C.c_uint64, [u8p, C.c_uint64, C.c_uint64]),
        "qzc_apply_gates_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, P(Gate),
                                           C.c_uint64]),
        "qzc_apply_gates_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, P(Gate),
                                          C.c_uint64]),
        "qzc_sim_create": (C.c_int, [C.c_void_p, P(SimConfig), P(C.c_void_p)]),
        "qzc_sim_destroy": (None, [C.c_void_p]),
        "qzc_sim_init_basis": (C.c_int, [C.c_void_p]),
        "qzc_sim_init_zero": (C.c_int, [C.c_void_p]),
        "qzc_exchange_pack_host": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, u32p, u32p, u8p, u32p,
                                             u32p, u8p, C.c_uint64, u64p]),
        "qzc_exchange_unpack_host": (C.c_int, [C.c_uint32, u8p, u64p, C.c_uint32, u8p, C.c_uint64, u32p,
                                               u32p]),
        "qzc_sim_run": (C.c_int, [C.c_void_p, P(Gate), C.c_uint64]),
        "qzc_sim_stats_get": (C.c_int, [C.c_void_p, P(SimStats)]),
        "qzc_sim_plan_stages": (C.c_int, [C.c_void_p, P(Gate), C.c_uint64, u64p]),
        "qzc_sim_digest": (C.c_int, [C.c_void_p, u64p]),
        "qzc_sim_norm": (C.c_int, [C.c_void_p, f64p]),
        "qzc_sim_chunk_count": (C.c_int, [C.c_void_p, u64p]),
        "qzc_sim_payload_bytes": (C.c_int, [C.c_void_p, u64p]),
        "qzc_sim_export": (C.c_int, [C.c_void_p, u8p, C.c_uint64, u32p, u32p]),
        "qzc_sim_import": (C.c_int, [C.c_void_p, u8p, u32p, u32p]),
        "qzc_sim_read_chunks": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
        "qzc_sim_write_chunk": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p]),
        "qzc_sim_fidelity_dev": (C.c_int, [C.c_void_p, C.c_void_p, f64p]),
        "qzc_dense_run": (C.c_int, [C.c_void_p, C.c_uint32, P(Gate), C.c_uint64,
                                    P(C.c_void_p)]),
        "qzc_dense_free": (None, [C.c_void_p, C.c_void_p]),
        "qzc_buffer_alloc": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_void_p)]),
        "qzc_buffer_free": (None, [C.c_void_p, C.c_void_p]),
        "qzc_copy_h2d": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]),
        "qzc_copy_d2h": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64]),
        "qzc_host_alloc": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_void_p)]),
        "qzc_host_free": (None, [C.c_void_p, C.c_void_p]),
        "qzc_pass_plan_stats": (C.c_int, [P(Gate), C.c_uint64, C.c_uint32, C.c_uint32, u64p]),
        "qzc_kprof_enable": (C.c_int, [C.c_void_p, C.c_int]),
        "qzc_sim_save": (C.c_int, [C.c_void_p, C.c_char_p]),
        "qzc_sim_load": (C.c_int, [C.c_void_p, C.c_char_p]),
        "qzc_sim_exchange_plan": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, u32p, u32p, u64p, u64p]),
        "qzc_sim_exchange_pack": (C.c_int, [C.c_void_p, P(C.c_void_p), u64p]),
        "qzc_sim_exchange_recv_buffer": (C.c_int, [C.c_void_p, C.c_uint64, P(C.c_void_p)]),
        "qzc_sim_exchange_unpack": (C.c_int, [C.c_void_p, u64p]),
        "qzc_kprof_read": (C.c_int, [C.c_void_p, P(KProfRecord), C.c_uint64, u64p]),
        "qzc_jit_wait": (C.c_uint64, []),
        "qzc_jit_selftest": (C.c_int, [P(Gate), C.c_uint64, C.c_uint32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    # specialised-pass compiles still running at interpreter exit would race
    # NVRTC's own teardown: let them finish first
    import atexit
    atexit.register(lib.qzc_jit_wait)
    return lib


def pass_plan_stats(gates, nbits: int, fuse="relaxed") -> dict:
    """Fused-pass plan summary for gates on buffer bits of a 2^nbits window
    (host-only planning, no GPU needed)."""
    lib = load_library()
    arr = to_array(gates)
    out = (C.c_uint64 * 6)()
    mode = {"none": 0, "relaxed": 1, "strict": 2, "checked": 3}[fuse]
    _check(lib.qzc_pass_plan_stats(arr.ctypes.data_as(P(Gate)), arr.size, nbits, mode, out))
    keys = ("passes", "groups", "relaxed_groups", "gates", "fast_ops", "pdiag_ops")
    return dict(zip(keys, (int(x) for x in out)))


def jit_selftest(gates, nbits: int) -> None:
    """Compile the widest fused pass of `gates` (on buffer bits of a 2^nbits
    window) as a runtime-specialised kernel with NVRTC (host only, no GPU);
    raises with NVRTC's log when the toolchain cannot build it."""
    lib = load_library()
    arr = to_array(gates)
    _check(lib.qzc_jit_selftest(arr.ctypes.data_as(P(Gate)), arr.size, nbits))


def jit_wait() -> int:
    """Block until every queued specialised-pass compile has finished
    (e.g. after a warm-up run); returns how many were built."""
    return int(load_library().qzc_jit_wait())


def exported_symbols() -> list[str]:
    """Names declared in include/qzcuda.h (for the load/export test)."""
    import re
    hdr = (Path(__file__).resolve().parents[1] / "include" / "qzcuda.h").read_text()
    return sorted(set(re.findall(r"\b(qzc_[a-z0-9_]+)\s*\(", hdr)))


def _check(rc: int) -> None:
    if rc != 0:
        msg = load_library().qzc_last_error().decode()
        raise _ERRORS.get(rc, QzError)(msg)


def _amps(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


class Engine:
    """One CUDA context (qzc_context) on one GPU."""

    def __init__(self, device: int = 0, hbm_budget: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        _check(self.lib.qzc_context_create(device, hbm_budget, C.byref(h)))
        self.h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.qzc_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.qzc_kernel_launches(self.h))

    def timer_begin(self) -> None:
        _check(self.lib.qzc_timer_begin(self.h))

    def timer_end(self) -> float:
        """Seconds between timer_begin and now, CUDA events on the engine stream."""
        out = C.c_double()
        _check(self.lib.qzc_timer_end(self.h, C.byref(out)))
        return out.value

    def kprof_enable(self, on: bool = True) -> None:
        """Per-launch CUDA-event timing of the engine's kernels (clears records)."""
        _check(self.lib.qzc_kprof_enable(self.h, 1 if on else 0))

    def kprof_read(self) -> list[dict]:
        """Timed launches since enable / the last read (synchronizes)."""
        n = C.c_uint64()
        _check(self.lib.qzc_kprof_read(self.h, None, 0, C.byref(n)))
        recs = (KProfRecord * max(1, n.value))()
        _check(self.lib.qzc_kprof_read(self.h, recs, n.value, C.byref(n)))
        return [{"name": r.name.decode(), "tag": r.tag, "stage": r.stage, "seconds": r.seconds,
                 "bytes": r.bytes} for r in recs[:n.value]]

    def pinned(self, nbytes: int, dtype=np.uint8) -> np.ndarray:
        """Page-locked host array (qzc_host_alloc), freed with the array."""
        h = C.c_void_p()
        _check(self.lib.qzc_host_alloc(self.h, max(int(nbytes), 1), C.byref(h)))
        count = max(int(nbytes), 1) // np.dtype(dtype).itemsize
        raw = (C.c_uint8 * max(int(nbytes), 1)).from_address(h.value)
        arr = np.frombuffer(raw, dtype=dtype, count=count)
        lib, eh, ptr = self.lib, self.h, h.value
        import weakref
        weakref.finalize(raw, lib.qzc_host_free, eh, C.c_void_p(ptr))
        return arr

    def host_link_gbps(self, nbytes: int = 1 << 30, reps: int = 5) -> dict:
        """Pinned cudaMemcpyAsync H2D / D2H bandwidth (the host-link roofline
        of the host-staged residency), CUDA-event timed, best of `reps`."""
        amps = nbytes // 16
        h, d = C.c_void_p(), C.c_void_p()
        _check(self.lib.qzc_host_alloc(self.h, nbytes, C.byref(h)))
        _check(self.lib.qzc_buffer_alloc(self.h, amps, C.byref(d)))
        try:
            out = {}
            for name, fn, args in (("h2d", self.lib.qzc_copy_h2d, (d, 0, h, amps)),
                                   ("d2h", self.lib.qzc_copy_d2h, (h, d, 0, amps))):
                best = 1e30
                for _ in range(reps):
                    self.timer_begin()
                    _check(fn(self.h, *args))
                    best = min(best, self.timer_end())
                out[name] = nbytes / best / 1e9
            return out
        finally:
            self.lib.qzc_buffer_free(self.h, d)
            self.lib.qzc_host_free(self.h, h)

    # ---- gates ---------------------------------------------------------------
    def gate_matrix(self, g) -> np.ndarray:
        arr = to_array([g])
        m = np.zeros(16, dtype=np.complex128)
        dim = C.c_uint32()
        _check(self.lib.qzc_gate_matrix(gate_ptr(arr), m.ctypes.data, C.byref(dim)))
        return m[: dim.value ** 2].reshape(dim.value, dim.value)

    def apply_gates(self, amps, gates) -> np.ndarray:
        a = _amps(amps).copy()
        nbits = int(a.size).bit_length() - 1
        if a.size != 1 << nbits:
            raise ValueError("buffer length must be a power of two")
        arr = to_array(gates)
        _check(self.lib.qzc_apply_gates_host(self.h, a.ctypes.data, nbits, gate_ptr(arr), arr.size))
        return a

    def apply_gates_dev(self, ptr: int, nbits: int, gates) -> None:
        arr = to_array(gates)
        _check(self.lib.qzc_apply_gates_dev(self.h, ptr, nbits, gate_ptr(arr), arr.size))

    # ---- codec -----------------------------------------------------------------
    def compress_many(self, chunks, eb: float, forced=()):
        """chunks: (count, N) complex array → list of (payload bytes, crc)."""
        a = _amps(chunks)
        if a.ndim == 1:
            a = a[None, :]
        count, n = a.shape
        forced = np.ascontiguousarray(np.asarray(forced, dtype=np.uint64))
        cap = int(self.lib.qzc_payload_bound(n, eb)) * count + 64
        out = np.zeros(cap, dtype=np.uint8)
        offs = np.zeros(count, dtype=np.uint64)
        sizes = np.zeros(count, dtype=np.uint32)
        crcs = np.zeros(count, dtype=np.uint32)
        _check(self.lib.qzc_compress_host(self.h, a.ctypes.data, count, n, eb,
                                          forced.ctypes.data_as(u64p), forced.size,
                                          out.ctypes.data_as(u8p), cap,
                                          offs.ctypes.data_as(u64p), sizes.ctypes.data_as(u32p),
                                          crcs.ctypes.data_as(u32p)))
        return [(out[int(o):int(o) + int(s)].tobytes(), int(c)) for o, s, c in zip(offs, sizes, crcs)]

    def compress(self, amps, eb: float, forced=()):
        return self.compress_many(_amps(amps)[None, :], eb, forced)[0]

    def decompress_many(self, payloads, crcs, n: int, chunk_index_base: int = 0) -> np.ndarray:
        blob = b"".join(payloads)
        buf = np.frombuffer(blob, dtype=np.uint8).copy() if blob else np.zeros(1, np.uint8)
        sizes = np.array([len(p) for p in payloads], dtype=np.uint32)
        offs = np.zeros(len(payloads), dtype=np.uint64)
        if len(payloads) > 1:
            offs[1:] = np.cumsum(sizes[:-1], dtype=np.uint64)
        crc = np.ascontiguousarray(np.asarray(crcs, dtype=np.uint32))
        out = np.zeros((len(payloads), n), dtype=np.complex128)
        _check(self.lib.qzc_decompress_host(self.h, buf.ctypes.data_as(u8p),
                                            offs.ctypes.data_as(u64p), sizes.ctypes.data_as(u32p),
                                            crc.ctypes.data_as(u32p), len(payloads), n,
                                            chunk_index_base, out.ctypes.data))
        return out

    def decompress(self, payload: bytes, crc: int, n: int, chunk_index: int = 0) -> np.ndarray:
        return self.decompress_many([payload], [crc], n, chunk_index)[0]

    # ---- simulator ---------------------------------------------------------------
    def simulator(self, n: int, c: int, m: int, eb: float, **kw) -> "Simulator":
        return Simulator(self, n, c, m, eb, **kw)

    def dense_state(self, n: int, gates) -> "DenseState":
        return DenseState(self, n, gates)


class DenseState:
    """Uncompressed fp64 state on the GPU (fidelity baseline)."""

    def __init__(self, eng: Engine, n: int, gates):
        self.eng, self.n = eng, n
        arr = to_array(gates)
        p = C.c_void_p()
        _check(eng.lib.qzc_dense_run(eng.h, n, gate_ptr(arr), arr.size, C.byref(p)))
        self.ptr = p

    def free(self) -> None:
        if self.ptr:
            self.eng.lib.qzc_dense_free(self.eng.h, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Simulator:
    """Compressed-chunk state vector in HBM (qzc_sim) — qzsim::run's hot path."""

    def __init__(self, eng: Engine, n: int, c: int, m: int, eb: float, window_amps: int = 0,
                 fuse=True, init: bool = True, residency: str = "hbm",
                 force_replay: bool = False, skip_reencode: bool = False):
        """fuse: True = fused passes with relaxed +0-safe diagonal units
        (default), "checked" = also checked diagonal units (out-of-place
        passes, per-pass replay), "strict" = every gate qubit in the tile,
        False = one pass per gate.  force_replay: always take the strict
        replay (test).  skip_reencode: NON-PARITY fast mode — one stage (one
        codec round trip) per run when the dense state fits HBM."""
        self.eng, self.lib = eng, eng.lib
        self.n, self.c, self.m, self.eb = n, c, m, eb
        cfg = SimConfig(num_qubits=n, chunk_qubits=c, batch_qubits=m, error_bound=eb,
                        window_amps=window_amps, residency={"hbm": 0, "host": 1}[residency],
                        renormalize=0,
                        fuse_gates={"strict": 2, "checked": 3}.get(fuse, 1 if fuse else 0),
                        debug_flags=1 if force_replay else 0,
                        skip_reencode=1 if skip_reencode else 0)
        h = C.c_void_p()
        _check(self.lib.qzc_sim_create(eng.h, C.byref(cfg), C.byref(h)))
        self.h = h
        if init:
            self.init_basis()

    def close(self) -> None:
        if getattr(self, "h", None):
            # (a simulator outliving its engine — interpreter teardown order —
            # is leaked rather than destroyed against a freed context)
            if getattr(self.eng, "h", None):
                self.lib.qzc_sim_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def chunk_count(self) -> int:
        return 1 << (self.n - self.c)

    def init_basis(self) -> None:
        _check(self.lib.qzc_sim_init_basis(self.h))

    def init_zero(self) -> None:
        """Every chunk the zero-chunk payload (non-zero ranks of a sharded |0...0>)."""
        _check(self.lib.qzc_sim_init_zero(self.h))

    def run(self, gates) -> None:
        arr = to_array(gates)
        _check(self.lib.qzc_sim_run(self.h, gate_ptr(arr), arr.size))

    def plan_stages(self, gates) -> int:
        arr = to_array(gates)
        out = C.c_uint64()
        _check(self.lib.qzc_sim_plan_stages(self.h, gate_ptr(arr), arr.size, C.byref(out)))
        return out.value

    def stats(self) -> dict:
        st = SimStats()
        _check(self.lib.qzc_sim_stats_get(self.h, C.byref(st)))
        d = st.as_dict()
        d["ratio"] = d["dense_bytes"] / d["current_bytes"] if d["current_bytes"] else 0.0
        return d

    def digest(self) -> int:
        out = C.c_uint64()
        _check(self.lib.qzc_sim_digest(self.h, C.byref(out)))
        return out.value

    def norm(self) -> float:
        out = C.c_double()
        _check(self.lib.qzc_sim_norm(self.h, C.byref(out)))
        return out.value

    def payload_bytes(self) -> int:
        out = C.c_uint64()
        _check(self.lib.qzc_sim_payload_bytes(self.h, C.byref(out)))
        return out.value

    def export(self, out=None, sizes=None, crcs=None):
        """The store's payloads in chunk order, sizes and CRCs.  Without `out`
        the payloads come back as bytes; with `out` (a writable uint8 array,
        e.g. Engine.pinned(...), reused across calls) they are written into it
        and a view of the used prefix is returned — no host-side copy."""
        total = self.payload_bytes()
        buf = np.empty(max(total, 1), dtype=np.uint8) if out is None else out
        if buf.size < total:
            raise ValueError(f"export buffer holds {buf.size} bytes, the store needs {total}")
        sizes = np.empty(self.chunk_count, dtype=np.uint32) if sizes is None else sizes
        crcs = np.empty(self.chunk_count, dtype=np.uint32) if crcs is None else crcs
        _check(self.lib.qzc_sim_export(self.h, buf.ctypes.data_as(u8p), buf.size,
                                       sizes.ctypes.data_as(u32p), crcs.ctypes.data_as(u32p)))
        return (buf[:total].tobytes() if out is None else buf[:total]), sizes, crcs

    def import_(self, payload: bytes, sizes, crcs) -> None:
        buf = np.frombuffer(payload, dtype=np.uint8).copy() if payload else np.zeros(1, np.uint8)
        sizes = np.ascontiguousarray(sizes, dtype=np.uint32)
        crcs = np.ascontiguousarray(crcs, dtype=np.uint32)
        _check(self.lib.qzc_sim_import(self.h, buf.ctypes.data_as(u8p),
                                       sizes.ctypes.data_as(u32p), crcs.ctypes.data_as(u32p)))

    def read_chunks(self, first: int = 0, count: int | None = None) -> np.ndarray:
        count = self.chunk_count - first if count is None else count
        out = np.zeros(count << self.c, dtype=np.complex128)
        _check(self.lib.qzc_sim_read_chunks(self.h, first, count, out.ctypes.data))
        return out

    def state(self) -> np.ndarray:
        return self.read_chunks(0, self.chunk_count)

    def write_chunk(self, index: int, amps) -> None:
        a = _amps(amps)
        if a.size != 1 << self.c:
            raise StoreError(f"chunk size mismatch: expected {1 << self.c}, got {a.size}")
        _check(self.lib.qzc_sim_write_chunk(self.h, index, a.ctypes.data))

    # ---- checkpoint / resume (ChunkStore::save / load, store.cpp:152-217) ----
    def save(self, path) -> None:
        """Write the store as a QZST file (the reference's format)."""
        _check(self.lib.qzc_sim_save(self.h, os.fsencode(str(path))))

    def load(self, path) -> None:
        """Replace the store with a QZST file's chunks (CRCs verified on the GPU)."""
        _check(self.lib.qzc_sim_load(self.h, os.fsencode(str(path))))

    # ---- sharded exchange (device to device; sharding.py drives it) --------
    def exchange_plan(self, g: int, rank: int, old_pos, new_pos):
        """Per-destination record-group bytes and chunk counts of an ownership
        change from owner positions old_pos to new_pos (chunk-index bits)."""
        world = 1 << g
        op = np.ascontiguousarray(old_pos, dtype=np.uint32)
        np_ = np.ascontiguousarray(new_pos, dtype=np.uint32)
        sb = np.zeros(world, np.uint64)
        sc = np.zeros(world, np.uint64)
        _check(self.lib.qzc_sim_exchange_plan(self.h, g, rank, op.ctypes.data_as(u32p),
                                              np_.ctypes.data_as(u32p), sb.ctypes.data_as(u64p),
                                              sc.ctypes.data_as(u64p)))
        return sb, sc

    def exchange_pack(self) -> tuple[int, int]:
        """Pack the planned groups in HBM: (device pointer, bytes)."""
        p, n = C.c_void_p(), C.c_uint64()
        _check(self.lib.qzc_sim_exchange_pack(self.h, C.byref(p), C.byref(n)))
        return int(p.value or 0), int(n.value)

    def exchange_recv_buffer(self, nbytes: int) -> int:
        p = C.c_void_p()
        _check(self.lib.qzc_sim_exchange_recv_buffer(self.h, int(nbytes), C.byref(p)))
        return int(p.value or 0)

    def exchange_unpack(self, recv_bytes) -> None:
        rb = np.ascontiguousarray(recv_bytes, dtype=np.uint64)
        _check(self.lib.qzc_sim_exchange_unpack(self.h, rb.ctypes.data_as(u64p)))

    def fidelity(self, dense: DenseState) -> float:
        out = C.c_double()
        _check(self.lib.qzc_sim_fidelity_dev(self.h, dense.ptr, C.byref(out)))
        return out.value
