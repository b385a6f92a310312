"""Sharded execution of the staged pipeline over G = 2^g GPUs.

Not in the reference (SPEC.md:192 lists distribution as a non-goal); this is
the north star's item 4 / SURVEY §5 and §8e:

* **Ownership.** Rank r owns every chunk whose bits at the g *owner* positions
  (chunk-index bits, i.e. qubits >= c) spell r.  A rank's chunks form an
  (n-g)-qubit compressed store of their own: local chunk index = global index
  with the owner bits squeezed out, local qubit label = global label minus
  the owner qubits below it.
* **Stages.** The global planner's stage partition is kept (one codec round
  trip per chunk per stage).  Owner qubits must not be touched
  by a stage's gates; each rank then runs the stage on its own store as one
  local stage (`Simulator.run` on the relabelled gates).  Batch membership
  differs from the single-GPU run only in padding, which never changes a
  payload byte, so the final store — and the FNV digest over chunks in
  global order — is identical to the reference's.
* **Exchange.** When a stage touches an owner qubit, that owner position is
  re-assigned to a free qubit (the one whose next use is farthest away) and
  whole *compressed* chunks move to their new owner: an all-to-all of
  (new local index, size, crc, payload) records.  Over NVLink this is NCCL
  all_to_all on the payload bytes; tests run it over gloo on CPU.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from .abi import gate_ptr, to_array


@dataclass
class StageInfo:
    first: int
    count: int
    high: list          # padded high set (global labels)
    touched: list       # qubits >= c used by the stage's gates


def global_stages(n: int, c: int, m: int, gates) -> list[StageInfo]:
    """The reference planner's stage partition (qzc_plan_export)."""
    from .engine import _check, load_library
    lib = load_library()
    arr = to_array(gates)
    cap = max(arr.size, 1)
    ns = C.c_uint64()
    first = np.zeros(cap, np.uint64)
    cnt = np.zeros(cap, np.uint64)
    nh = np.zeros(cap, np.uint32)
    hi = np.zeros(64 * cap, np.uint32)
    P = C.POINTER
    lib.qzc_plan_export.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64,
                                    P(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_uint64]
    _check(lib.qzc_plan_export(n, c, m, arr.ctypes.data, arr.size, C.byref(ns), first.ctypes.data,
                               cnt.ctypes.data, nh.ctypes.data, hi.ctypes.data, cap))
    out = []
    for s in range(ns.value):
        f, k = int(first[s]), int(cnt[s])
        touched = sorted({int(q) for g in arr[f:f + k] for q in g["qubits"][: int(g["nqubits"])]
                          if q >= c})
        out.append(StageInfo(f, k, [int(x) for x in hi[64 * s: 64 * s + nh[s]]], touched))
    return out


def plan_owners(n: int, c: int, g: int, stages: list[StageInfo]) -> list[list[int]]:
    """Owner qubits per stage (position i = rank bit i).  Initially the top g
    qubits; an owner touched by a stage is replaced by the free qubit whose
    next use is farthest in the future (ties: higher qubit)."""
    if g == 0:
        return [[] for _ in stages]
    if n - g < c + 2:
        raise ValueError(f"cannot shard {n} qubits over 2^{g} ranks with c={c}")
    owners = list(range(n - g, n))
    plans = []
    for si, st in enumerate(stages):
        touched = set(st.touched)
        if len(touched) > (n - c) - g:
            raise ValueError(f"stage {si} touches {len(touched)} high qubits; at most "
                             f"{n - c - g} can stay local with {2 ** g} ranks")

        def next_use(q):
            for sj in range(si, len(stages)):
                if q in stages[sj].touched:
                    return sj
            return len(stages) + 1

        for i, q in enumerate(owners):
            if q in touched:
                free = [x for x in range(c, n) if x not in touched and x not in owners]
                best = max(free, key=lambda x: (next_use(x), x))
                owners[i] = best
        plans.append(list(owners))
    return plans


def _positions(owners, c):
    return [q - c for q in owners]


def squeeze(x: int, pos) -> int:
    """Remove the bits at `pos` from x."""
    out, j = 0, 0
    b = 0
    while x >> b:
        if b not in pos:
            out |= ((x >> b) & 1) << j
            j += 1
        b += 1
    return out


def expand(y: int, pos, rank: int) -> int:
    """Inverse of squeeze: bit i of `rank` goes to position pos[i], the bits
    of y fill the other positions in order."""
    taken = {p: i for i, p in enumerate(pos)}
    top = max(list(pos) + [0]) + 1 + y.bit_length()
    out, j = 0, 0
    for b in range(top + 1):
        if b in taken:
            out |= ((rank >> taken[b]) & 1) << b
        else:
            out |= ((y >> j) & 1) << b
            j += 1
    return out


def owner_of(x: int, pos) -> int:
    return sum(((x >> p) & 1) << i for i, p in enumerate(pos))


def local_gates(gates, owners, c):
    """Relabel a stage's gates to the rank-local (n-g)-qubit register."""
    arr = to_array(gates).copy()
    ow = sorted(owners)
    for gt in arr:
        for k in range(int(gt["nqubits"])):
            q = int(gt["qubits"][k])
            assert q not in ow, "stage touches an owner qubit"
            gt["qubits"][k] = q - sum(1 for o in ow if o < q)
    return arr


def pack_records(records) -> bytes:
    """(new_local_index, crc, payload) -> bytes"""
    out = bytearray()
    for idx, crc, payload in records:
        out += struct.pack("<QII", idx, len(payload), crc) + payload
    return bytes(out)


def unpack_records(blob: bytes):
    out, pos = [], 0
    while pos < len(blob):
        idx, size, crc = struct.unpack_from("<QII", blob, pos)
        pos += 16
        out.append((idx, crc, blob[pos:pos + size]))
        pos += size
    return out


def exchange_plan(store_blob: bytes, sizes, crcs, rank: int, old_owners, new_owners, c, world):
    """Split this rank's exported store into per-destination record lists."""
    old_pos, new_pos = _positions(old_owners, c), _positions(new_owners, c)
    per_dest = [[] for _ in range(world)]
    off = 0
    for y, (sz, crc) in enumerate(zip(sizes, crcs)):
        x = expand(y, old_pos, rank)
        dst = owner_of(x, new_pos)
        per_dest[dst].append((squeeze(x, new_pos), int(crc), store_blob[off:off + int(sz)]))
        off += int(sz)
    return per_dest


def assemble_store(records, nlocal):
    """Records (any order) -> (blob, sizes, crcs) in local chunk order."""
    recs = sorted(records, key=lambda r: r[0])
    assert [r[0] for r in recs] == list(range(nlocal)), "exchange lost or duplicated chunks"
    blob = b"".join(r[2] for r in recs)
    sizes = np.array([len(r[2]) for r in recs], np.uint32)
    crcs = np.array([r[1] for r in recs], np.uint32)
    return blob, sizes, crcs


class LocalGroup:
    """In-process transport: G ranks driven by one process (one GPU)."""

    def __init__(self, world: int):
        self.world = world

    def all_to_all(self, sends):
        # sends[r][d] -> recvs[d][r]
        return [[sends[r][d] for r in range(self.world)] for d in range(self.world)]


class TorchGroup:
    """torch.distributed transport (gloo on CPU, NCCL over NVLink)."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.device = device

    def all_to_all_bytes(self, send: list[bytes]) -> list[bytes]:
        import torch
        dev = self.device or "cpu"
        lens = torch.tensor([len(b) for b in send], dtype=torch.int64, device=dev)
        rlens = torch.empty_like(lens)
        self.dist.all_to_all_single(rlens, lens)
        flat = torch.frombuffer(bytearray(b"".join(send)) or bytearray(1), dtype=torch.uint8)
        if sum(len(b) for b in send) == 0:
            flat = flat[:0]
        flat = flat.to(dev)
        out = torch.empty(int(rlens.sum()), dtype=torch.uint8, device=dev)
        self.dist.all_to_all_single(out, flat, output_split_sizes=rlens.tolist(),
                                    input_split_sizes=lens.tolist())
        data = out.cpu().numpy().tobytes()
        res, pos = [], 0
        for k in rlens.tolist():
            res.append(data[pos:pos + k])
            pos += k
        return res


class ShardedRun:
    """Drive per-rank simulators through the sharded stage loop.

    `sims` are this process's rank simulators: one (torch.distributed, one
    process per GPU) or all G (LocalGroup, several ranks on one GPU)."""

    def __init__(self, engine_or_engines, n, c, m, eb, g, ranks, transport, **sim_kw):
        self.n, self.c, self.m, self.eb, self.g = n, c, m, eb, g
        self.world = 1 << g
        self.ranks = list(ranks)
        self.t = transport
        engs = engine_or_engines if isinstance(engine_or_engines, list) else \
            [engine_or_engines] * len(self.ranks)
        self.nl = n - g
        if self.nl < m:
            raise ValueError(f"local register {self.nl} qubits < batch qubits m={m}")
        self.sims = {r: e.simulator(self.nl, c, m, eb, init=False, **sim_kw)
                     for r, e in zip(self.ranks, engs)}
        self.engines = dict(zip(self.ranks, engs))
        self.owners = list(range(n - g, n))
        self.exchanges = 0
        self.exchanged_bytes = 0

    def init_basis(self):
        """|0...0>: rank 0 holds the basis chunk, all other ranks zeros."""
        for r, sim in self.sims.items():
            sim.init_basis()
            if r != 0:
                blob, sizes, crcs = sim.export()
                zero_payload, zcrc = self.engines[r].compress(
                    np.zeros(1 << self.c, np.complex128), self.eb)
                k = sim.chunk_count
                sim.import_(zero_payload * k, np.full(k, len(zero_payload), np.uint32),
                            np.full(k, zcrc, np.uint32))

    def _exchange(self, new_owners):
        sends = {}
        for r, sim in self.sims.items():
            blob, sizes, crcs = sim.export()
            per = exchange_plan(blob, sizes, crcs, r, self.owners, new_owners, self.c, self.world)
            sends[r] = [pack_records(p) for p in per]
        if isinstance(self.t, LocalGroup):
            recv = self.t.all_to_all([sends[r] for r in range(self.world)])
            recv = {r: recv[r] for r in self.ranks}
        else:
            (r,) = self.ranks
            recv = {r: self.t.all_to_all_bytes(sends[r])}
        nlocal = 1 << (self.nl - self.c)
        for r, sim in self.sims.items():
            self.exchanged_bytes += sum(len(b) for b in recv[r])
            recs = [rec for b in recv[r] for rec in unpack_records(b)]
            sim.import_(*assemble_store(recs, nlocal))
        self.owners = list(new_owners)
        self.exchanges += 1

    def run(self, gates):
        arr = to_array(gates)
        stages = global_stages(self.n, self.c, self.m, arr)
        plan = plan_owners(self.n, self.c, self.g, stages)
        for st, owners in zip(stages, plan):
            if owners != self.owners:
                self._exchange(owners)
            lg = local_gates(arr[st.first:st.first + st.count], self.owners, self.c)
            for sim in self.sims.values():
                sim.run(lg)

    def global_store(self):
        """(blob, sizes, crcs) of the whole state in global chunk order
        (ranks of this process only; LocalGroup holds all of them)."""
        pos = _positions(self.owners, self.c)
        recs = []
        for r, sim in self.sims.items():
            blob, sizes, crcs = sim.export()
            off = 0
            for y, (sz, crc) in enumerate(zip(sizes, crcs)):
                recs.append((expand(y, pos, r), int(crc), blob[off:off + int(sz)]))
                off += int(sz)
        return recs

    def gather_store(self):
        """All ranks' chunks at rank 0 (global order); None elsewhere."""
        recs = self.global_store()
        if isinstance(self.t, LocalGroup):
            return sorted(recs, key=lambda r: r[0])
        send = [b""] * self.world
        send[0] = pack_records(recs)
        got = self.t.all_to_all_bytes(send)
        if self.ranks[0] != 0:
            return None
        return sorted([r for b in got for r in unpack_records(b)], key=lambda r: r[0])

    def digest(self):
        """FNV-1a over all payloads in global chunk order (rank 0; None elsewhere)."""
        from .engine import load_library
        lib = load_library()
        recs = self.gather_store()
        if recs is None:
            return None
        h = 0xcbf29ce484222325
        for _, _, p in recs:
            buf = np.frombuffer(p, np.uint8).copy() if p else np.zeros(1, np.uint8)
            h = lib.qzc_fnv1a64(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(p), h)
        return h
