"""ctypes mirror of the plain-C types in include/qzcuda.h.

Shared by the product binding (``paper_2309_16979_b200.engine``) and the test
harness.  No behaviour lives here, only struct layouts and gate helpers.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

# Gate kinds, reference enum order (include/qzsim/gates.hpp:27-45).
KINDS = ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "rx", "ry", "rz", "u1",
         "u2", "u3", "cx", "cz", "swap"]
KIND = {name: i for i, name in enumerate(KINDS)}
ARITY = {k: (2 if k in ("cx", "cz", "swap") else 1) for k in KINDS}
NPARAMS = {k: {"rx": 1, "ry": 1, "rz": 1, "u1": 1, "u2": 2, "u3": 3}.get(k, 0)
           for k in KINDS}


class Gate(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("nqubits", C.c_uint32),
                ("qubits", C.c_uint32 * 2), ("params", C.c_double * 3)]


GATE_DTYPE = np.dtype([("kind", "<u4"), ("nqubits", "<u4"), ("qubits", "<u4", 2),
                       ("params", "<f8", 3)])
assert GATE_DTYPE.itemsize == C.sizeof(Gate) == 40


def gate(name: str, *qubits: int, params=()) -> tuple:
    name = name.lower()
    if len(qubits) != ARITY[name] or len(params) != NPARAMS[name]:
        raise ValueError(f"bad gate {name}{qubits}{params}")
    return (name, tuple(int(q) for q in qubits), tuple(float(p) for p in params))


def to_array(gates) -> np.ndarray:
    """List of (name, qubits, params) tuples or a GATE_DTYPE array → array."""
    if isinstance(gates, np.ndarray) and gates.dtype == GATE_DTYPE:
        return np.ascontiguousarray(gates)
    arr = np.zeros(len(gates), dtype=GATE_DTYPE)
    for i, (name, qs, ps) in enumerate(gates):
        arr[i]["kind"] = KIND[name]
        arr[i]["nqubits"] = len(qs)
        arr[i]["qubits"][: len(qs)] = qs
        arr[i]["params"][: len(ps)] = ps
    return arr


def from_array(arr: np.ndarray) -> list:
    out = []
    for g in arr:
        name = KINDS[int(g["kind"])]
        nq = int(g["nqubits"])
        out.append((name, tuple(int(q) for q in g["qubits"][:nq]),
                    tuple(float(p) for p in g["params"][:NPARAMS[name]])))
    return out


def gate_ptr(arr: np.ndarray):
    return arr.ctypes.data_as(C.POINTER(Gate))


class SimConfig(C.Structure):
    _fields_ = [("num_qubits", C.c_uint32), ("chunk_qubits", C.c_uint32),
                ("batch_qubits", C.c_uint32), ("skip_reencode", C.c_uint32),
                ("error_bound", C.c_double), ("window_amps", C.c_uint64),
                ("residency", C.c_uint32), ("renormalize", C.c_uint32),
                ("fuse_gates", C.c_uint32), ("debug_flags", C.c_uint32)]


class SimStats(C.Structure):
    _fields_ = [(name, C.c_double) for name in
                ("wall_seconds", "decode_seconds", "gate_seconds", "encode_seconds",
                 "h2d_seconds", "d2h_seconds")] + \
               [(name, C.c_uint64) for name in
                ("stages", "batches", "gate_passes", "chunk_decompress_count",
                 "chunk_recompress_count", "h2d_bytes", "d2h_bytes", "kernel_launches",
                 "current_bytes", "peak_bytes", "dense_bytes", "windows", "replays",
                 "payload_in_bytes", "payload_out_bytes")]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class KProfRecord(C.Structure):
    """qzc_kprof_record: one timed kernel launch."""
    _fields_ = [("name", C.c_char * 32), ("tag", C.c_uint32), ("stage", C.c_uint32),
                ("seconds", C.c_double), ("bytes", C.c_double)]

