"""Host-side logic of the sharded pipeline (paper_2309_16979_b200/sharding.py
and the engine's exchange record layout, csrc/qz_store_io.cu): ownership
planning, index squeeze/expand, and the chunk exchange — groups packed and
unpacked by the engine's host helpers (qzc_exchange_pack_host /
unpack_host: the same index math and format the device pack / unpack
kernels use) moved in-process and over torch.distributed gloo with
world_size 2 (CPU).  The device path itself runs in tests/test_gpu_shard.py."""
import os
import random

import numpy as np
import pytest

from paper_2309_16979_b200 import sharding as S
from paper_2309_16979_b200.sharding import StageInfo


def test_squeeze_expand_roundtrip():
    rng = random.Random(1)
    for _ in range(2000):
        nbits = rng.randint(2, 20)
        g = rng.randint(0, min(3, nbits - 1))
        pos = sorted(rng.sample(range(nbits), g))
        x = rng.randrange(1 << nbits)
        y = S.squeeze(x, pos)
        r = S.owner_of(x, pos)
        assert S.expand(y, pos, r) == x
        assert y < (1 << (nbits - g))


def test_expand_many_matches_expand():
    rng = random.Random(3)
    for _ in range(50):
        width = rng.randint(3, 16)
        g = rng.randint(1, 3)
        pos = rng.sample(range(width), g)
        rank = rng.randrange(1 << g)
        ys = np.arange(1 << (width - g), dtype=np.uint64)
        got = S.expand_many(ys, pos, rank, width)
        assert got.tolist() == [S.expand(int(y), pos, rank) for y in ys]


def test_plan_owners_never_touched_and_minimal():
    rng = random.Random(2)
    n, c = 14, 4
    for g in (1, 2, 3):
        stages = []
        for i in range(40):
            k = rng.randint(1, n - c - g)
            stages.append(StageInfo(i, 1, [], sorted(rng.sample(range(c, n), k))))
        plan = S.plan_owners(n, c, g, stages)
        prev = list(range(n - g, n))
        for st, ow in zip(stages, plan):
            assert len(set(ow)) == g and all(c <= q < n for q in ow)
            assert not set(ow) & set(st.touched)
            # only positions whose owner was touched change
            for i, (a, b) in enumerate(zip(prev, ow)):
                assert a == b or a in st.touched
            prev = ow


def _mock_store(nl_chunks, rank, owners, c, seed=0):
    """payload bytes encode the global chunk index -> exchange is checkable"""
    pos = S.positions(owners, c)
    blobs, sizes, crcs = [], [], []
    for y in range(nl_chunks):
        x = S.expand(y, pos, rank)
        p = x.to_bytes(8, "little") * (1 + (x * 7 + seed) % 5) + bytes([seed % 7] * (x % 3))
        blobs.append(p)
        sizes.append(len(p))
        crcs.append(x & 0xffffffff)
    return b"".join(blobs), np.array(sizes, np.uint32), np.array(crcs, np.uint32)


def _check_store(blob, sizes, crcs, rank, owners, c):
    pos = S.positions(owners, c)
    off = 0
    for y, sz in enumerate(sizes):
        x = S.expand(y, pos, rank)
        p = blob[off:off + int(sz)]
        off += int(sz)
        assert p[:8] == x.to_bytes(8, "little")
        assert int(crcs[y]) == x & 0xffffffff


def _exchange_host(stores, world, g, local_bits, owners, new, c):
    groups = {r: S.pack_groups_host(local_bits, g, r, S.positions(owners, c), S.positions(new, c),
                                    *stores[r]) for r in range(world)}
    out = {}
    for d in range(world):
        parts, rb = [], []
        for s in range(world):
            buf, sb = groups[s]
            o = int(sb[:d].sum())
            parts.append(buf[o:o + int(sb[d])])
            rb.append(int(sb[d]))
        out[d] = S.unpack_groups_host(world, b"".join(parts), rb, local_bits)
    return out


@pytest.mark.parametrize("g", [1, 2, 3])
def test_host_layout_exchange(g):
    n, c = 12, 3
    world = 1 << g
    local_bits = n - c - g
    owners = list(range(n - g, n))
    stores = {r: _mock_store(1 << local_bits, r, owners, c) for r in range(world)}
    rng = random.Random(g)
    for _ in range(6):
        new = list(owners)
        i = rng.randrange(g)
        new[i] = rng.choice([q for q in range(c, n) if q not in owners])
        stores = _exchange_host(stores, world, g, local_bits, owners, new, c)
        owners = new
        for r in range(world):
            _check_store(*stores[r], r, owners, c)


def test_group_layout_is_16_byte_aligned_and_sized():
    n, c, g = 10, 2, 2
    local_bits = n - c - g
    owners = list(range(n - g, n))
    store = _mock_store(1 << local_bits, 1, owners, c)
    buf, sb = S.pack_groups_host(local_bits, g, 1, S.positions(owners, c), S.positions([3, 9], c), *store)
    assert all(int(x) % 16 == 0 for x in sb) and len(buf) == int(sb.sum())
    # every chunk lands in exactly one group; group d holds the chunks whose
    # new owner bits spell d
    counts = [int.from_bytes(buf[int(sb[:d].sum()):int(sb[:d].sum()) + 8], "little")
              for d in range(1 << g)]
    assert sum(counts) == 1 << local_bits


def test_unpack_rejects_missing_and_duplicate_chunks():
    from paper_2309_16979_b200 import engine as E
    n, c, g = 9, 2, 1
    local_bits = n - c - g
    owners = [n - 1]
    store = _mock_store(1 << local_bits, 0, owners, c)
    buf, sb = S.pack_groups_host(local_bits, g, 0, S.positions(owners, c), S.positions([c], c), *store)
    assert int(sb[0]) and int(sb[1])
    # only this rank's own group: half of the chunks are missing
    with pytest.raises(E.StoreError):
        S.unpack_groups_host(2, buf[:int(sb[0])], [int(sb[0]), 0], local_bits)
    # the same group twice: duplicates
    with pytest.raises(E.StoreError):
        S.unpack_groups_host(2, buf[:int(sb[0])] * 2, [int(sb[0]), int(sb[0])], local_bits)


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, c = 11, 3
        g = world.bit_length() - 1
        local_bits = n - c - g
        owners = list(range(n - g, n))
        store = _mock_store(1 << local_bits, rank, owners, c, seed=5)
        for new_q in (4, 6, 9, 5):
            new = [new_q] + owners[1:] if new_q not in owners else owners
            buf, sb = S.pack_groups_host(local_bits, g, rank, S.positions(owners, c),
                                         S.positions(new, c), *store)
            send_sizes = torch.tensor(sb.astype(np.int64))
            recv_sizes = torch.empty_like(send_sizes)
            dist.all_to_all_single(recv_sizes, send_sizes)
            rb = recv_sizes.numpy()
            recv = torch.empty(int(rb.sum()), dtype=torch.uint8)
            dist.all_to_all_single(recv, torch.frombuffer(bytearray(buf), dtype=torch.uint8),
                                   [int(x) for x in rb], [int(x) for x in sb])
            store = S.unpack_groups_host(world, recv.numpy().tobytes(), rb, local_bits)
            owners = new
            _check_store(*store, rank, owners, c)
        out.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        out.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}
