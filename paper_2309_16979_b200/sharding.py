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
  whole *compressed* chunks move to their new owner, device to device: the
  engine packs per-destination record groups in HBM from the arena
  (qzc_sim_exchange_plan / _pack), the transport moves them (NCCL
  all_to_all over NVLink; gloo through host memory in the CPU-backed
  tests), and the engine unpacks the received groups in place — the receive
  buffer becomes the new arena (qzc_sim_exchange_unpack).  Only the group
  sizes (2^g integers) cross the host.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .abi import to_array


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


def positions(owners, c) -> list[int]:
    """Owner qubits -> chunk-index bit positions."""
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


def expand_many(ys: np.ndarray, pos, rank: int, width: int) -> np.ndarray:
    """Vectorised expand over local chunk indices (width = global index bits)."""
    ys = np.asarray(ys, dtype=np.uint64)
    x = np.zeros_like(ys)
    taken = {p: i for i, p in enumerate(pos)}
    j = 0
    for b in range(width):
        if b in taken:
            if (rank >> taken[b]) & 1:
                x |= np.uint64(1 << b)
        else:
            x |= ((ys >> np.uint64(j)) & np.uint64(1)) << np.uint64(b)
            j += 1
    return x


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


# ------------------------------------------------------------------ host path
def pack_groups_host(local_bits: int, g: int, rank: int, old_pos, new_pos, blob: bytes, sizes,
                     crcs) -> tuple[bytes, np.ndarray]:
    """The engine's record groups built on the host from a store given as
    payloads in local chunk order (qzc_exchange_pack_host): (buffer, bytes per
    destination).  Same layout the device pack writes."""
    from .engine import _check, load_library
    lib = load_library()
    P = C.POINTER
    op = np.ascontiguousarray(old_pos, np.uint32)
    np_ = np.ascontiguousarray(new_pos, np.uint32)
    sizes = np.ascontiguousarray(sizes, np.uint32)
    crcs = np.ascontiguousarray(crcs, np.uint32)
    payload = np.frombuffer(blob, np.uint8) if blob else np.zeros(1, np.uint8)
    sb = np.zeros(1 << g, np.uint64)
    args = (local_bits, g, rank, op.ctypes.data_as(P(C.c_uint32)), np_.ctypes.data_as(P(C.c_uint32)),
            payload.ctypes.data_as(P(C.c_uint8)), sizes.ctypes.data_as(P(C.c_uint32)),
            crcs.ctypes.data_as(P(C.c_uint32)))
    _check(lib.qzc_exchange_pack_host(*args, None, 0, sb.ctypes.data_as(P(C.c_uint64))))
    out = np.zeros(max(int(sb.sum()), 1), np.uint8)
    _check(lib.qzc_exchange_pack_host(*args, out.ctypes.data_as(P(C.c_uint8)), out.size,
                                      sb.ctypes.data_as(P(C.c_uint64))))
    return out[: int(sb.sum())].tobytes(), sb


def unpack_groups_host(world: int, recv: bytes, recv_bytes, local_bits: int):
    """Received groups -> (blob, sizes, crcs) in local chunk order
    (qzc_exchange_unpack_host)."""
    from .engine import _check, load_library
    lib = load_library()
    P = C.POINTER
    buf = np.frombuffer(recv, np.uint8) if recv else np.zeros(1, np.uint8)
    rb = np.ascontiguousarray(recv_bytes, np.uint64)
    n = 1 << local_bits
    sizes = np.zeros(n, np.uint32)
    crcs = np.zeros(n, np.uint32)
    out = np.zeros(max(len(recv), 1), np.uint8)
    _check(lib.qzc_exchange_unpack_host(world, buf.ctypes.data_as(P(C.c_uint8)),
                                        rb.ctypes.data_as(P(C.c_uint64)), local_bits,
                                        out.ctypes.data_as(P(C.c_uint8)), out.size,
                                        sizes.ctypes.data_as(P(C.c_uint32)),
                                        crcs.ctypes.data_as(P(C.c_uint32))))
    return out[: int(sizes.sum(dtype=np.uint64))].tobytes(), sizes, crcs


# ---------------------------------------------------------------- transports
class _DevBytes:
    """Zero-copy __cuda_array_interface__ view of an engine device buffer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_view(ptr: int, nbytes: int, device):
    import torch
    if nbytes == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_DevBytes(ptr, nbytes), device=device)


class LocalGroup:
    """In-process transport: G ranks driven by one process (one GPU); the
    groups move with device-to-device copies."""

    def __init__(self, world: int):
        self.world = world

    def exchange(self, sims: dict, plans: dict, device) -> int:
        import torch
        sends = {r: sims[r].exchange_pack() for r in sims}
        moved = 0
        recv_bytes = {}
        for d in range(self.world):
            rb = np.array([int(plans[s][d]) for s in range(self.world)], np.uint64)
            rptr = sims[d].exchange_recv_buffer(int(rb.sum()))
            dst_off = 0
            for s in range(self.world):
                sptr, _ = sends[s]
                src_off = int(plans[s][:d].sum())
                n = int(plans[s][d])
                if n:
                    device_view(rptr + dst_off, n, device).copy_(device_view(sptr + src_off, n, device))
                dst_off += n
                moved += n if s != d else 0
            recv_bytes[d] = rb
        torch.cuda.synchronize(device)
        for d in range(self.world):
            sims[d].exchange_unpack(recv_bytes[d])
        return moved

    def allgather_bytes(self, payloads: dict) -> dict:
        return payloads


class TorchGroup:
    """torch.distributed transport: NCCL moves the groups GPU to GPU; gloo
    (CPU-backed tests) stages them through host memory."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.device = device
        self.nccl = dist.get_backend() == "nccl"

    def exchange(self, sims: dict, plans: dict, device) -> int:
        import torch
        (r,) = sims
        sim = sims[r]
        sb = plans[r]
        cdev = device if self.nccl else "cpu"
        send_sizes = torch.tensor(sb.astype(np.int64), device=cdev)
        recv_sizes = torch.empty_like(send_sizes)
        self.dist.all_to_all_single(recv_sizes, send_sizes)
        rb = recv_sizes.cpu().numpy().astype(np.uint64)
        sptr, total = sim.exchange_pack()
        rptr = sim.exchange_recv_buffer(int(rb.sum()))
        send = device_view(sptr, total, device)
        recv = device_view(rptr, int(rb.sum()), device)
        if self.nccl:
            self.dist.all_to_all_single(recv, send, [int(x) for x in rb], [int(x) for x in sb])
            torch.cuda.synchronize(device)
        else:
            rcpu = torch.empty(int(rb.sum()), dtype=torch.uint8)
            self.dist.all_to_all_single(rcpu, send.cpu(), [int(x) for x in rb], [int(x) for x in sb])
            recv.copy_(rcpu.to(device))
            torch.cuda.synchronize(device)
        sim.exchange_unpack(rb)
        return int(sb.sum() - sb[r])

    def all_to_all_bytes(self, send: list[bytes]) -> list[bytes]:
        """Host byte strings to every rank (report path: digest gathering)."""
        import torch
        dev = self.device if self.nccl else "cpu"
        lens = torch.tensor([len(b) for b in send], dtype=torch.int64, device=dev)
        rlens = torch.empty_like(lens)
        self.dist.all_to_all_single(rlens, lens)
        joined = b"".join(send)
        flat = torch.frombuffer(bytearray(joined), dtype=torch.uint8) if joined else \
            torch.empty(0, dtype=torch.uint8)
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
        self.device = f"cuda:{engs[0].device}"
        self.owners = list(range(n - g, n))
        self.exchanges = 0
        self.exchanged_bytes = 0

    def init_basis(self):
        """|0...0>: rank 0 holds the basis chunk, all other ranks zeros."""
        self.owners = list(range(self.n - self.g, self.n))
        for r, sim in self.sims.items():
            if r == 0:
                sim.init_basis()
            else:
                sim.init_zero()

    def _exchange(self, new_owners):
        old_pos, new_pos = positions(self.owners, self.c), positions(new_owners, self.c)
        plans = {r: sim.exchange_plan(self.g, r, old_pos, new_pos)[0] for r, sim in self.sims.items()}
        self.exchanged_bytes += self.t.exchange(self.sims, plans, self.device)
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

    def local_export(self):
        """This process's rank stores on the host: {rank: (blob, sizes, crcs)}."""
        return {r: sim.export() for r, sim in self.sims.items()}

    def global_chunk_indices(self, rank: int) -> np.ndarray:
        nloc = 1 << (self.nl - self.c)
        return expand_many(np.arange(nloc, dtype=np.uint64), positions(self.owners, self.c), rank,
                           self.n - self.c)

    def gather_store(self):
        """All chunks at rank 0 in global chunk order: (blob, sizes, crcs);
        None on the other ranks (report path, not timed)."""
        import struct
        parts = {}
        for r, (blob, sizes, crcs) in self.local_export().items():
            parts[r] = (self.global_chunk_indices(r), blob, sizes, crcs)
        if not isinstance(self.t, LocalGroup):
            (r,) = self.ranks
            idx, blob, sizes, crcs = parts[r]
            msg = struct.pack("<QQ", r, len(idx)) + idx.tobytes() + sizes.tobytes() + \
                crcs.tobytes() + blob
            send = [b""] * self.world
            send[0] = msg
            got = self.t.all_to_all_bytes(send)
            if r != 0:
                return None
            parts = {}
            for m_ in got:
                src, k = struct.unpack_from("<QQ", m_, 0)
                o = 16
                idx = np.frombuffer(m_, np.uint64, k, o)
                o += 8 * k
                sizes = np.frombuffer(m_, np.uint32, k, o)
                o += 4 * k
                crcs = np.frombuffer(m_, np.uint32, k, o)
                o += 4 * k
                parts[src] = (idx, m_[o:], sizes, crcs)
        total = 1 << (self.n - self.c)
        sizes_g = np.zeros(total, np.uint32)
        crcs_g = np.zeros(total, np.uint32)
        chunks = [b""] * total
        for idx, blob, sizes, crcs in parts.values():
            offs = np.concatenate([[0], np.cumsum(sizes, dtype=np.uint64)]).astype(np.int64)
            for j, x in enumerate(idx.tolist()):
                chunks[x] = bytes(blob[offs[j]:offs[j + 1]])
            sizes_g[idx.astype(np.int64)] = sizes
            crcs_g[idx.astype(np.int64)] = crcs
        return b"".join(chunks), sizes_g, crcs_g

    def digest(self):
        """FNV-1a over all payloads in global chunk order (rank 0; None elsewhere)."""
        from .engine import load_library
        g = self.gather_store()
        if g is None:
            return None
        blob = g[0]
        buf = np.frombuffer(blob, np.uint8) if blob else np.zeros(1, np.uint8)
        return load_library().qzc_fnv1a64(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(blob),
                                          0xcbf29ce484222325)
