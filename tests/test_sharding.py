"""Host-side logic of the sharded pipeline (paper_2309_16979_b200/sharding.py):
ownership planning, index squeeze/expand, the chunk exchange over an
in-process group and over torch.distributed gloo with world_size 2 (CPU)."""
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
    pos = [q - c for q in owners]
    blobs, sizes, crcs = [], [], []
    for y in range(nl_chunks):
        x = S.expand(y, pos, rank)
        p = x.to_bytes(8, "little") * (1 + (x * 7 + seed) % 5)
        blobs.append(p)
        sizes.append(len(p))
        crcs.append(x & 0xffffffff)
    return b"".join(blobs), np.array(sizes, np.uint32), np.array(crcs, np.uint32)


def _check_store(blob, sizes, crcs, rank, owners, c):
    pos = [q - c for q in owners]
    off = 0
    for y, sz in enumerate(sizes):
        x = S.expand(y, pos, rank)
        p = blob[off:off + int(sz)]
        off += int(sz)
        assert p[:8] == x.to_bytes(8, "little")
        assert int(crcs[y]) == x & 0xffffffff


@pytest.mark.parametrize("g", [1, 2, 3])
def test_local_group_exchange(g):
    n, c = 12, 3
    world = 1 << g
    nl = 1 << (n - c - g)
    owners = list(range(n - g, n))
    stores = {r: _mock_store(nl, r, owners, c) for r in range(world)}
    grp = S.LocalGroup(world)
    rng = random.Random(g)
    for _ in range(6):
        new = list(owners)
        i = rng.randrange(g)
        new[i] = rng.choice([q for q in range(c, n) if q not in owners])
        sends = [[S.pack_records(p) for p in S.exchange_plan(*stores[r], r, owners, new, c, world)]
                 for r in range(world)]
        recv = grp.all_to_all(sends)
        stores = {r: S.assemble_store([rec for b in recv[r] for rec in S.unpack_records(b)], nl)
                  for r in range(world)}
        owners = new
        for r in range(world):
            _check_store(*stores[r], r, owners, c)


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, c = 11, 3
        g = world.bit_length() - 1
        nl = 1 << (n - c - g)
        owners = list(range(n - g, n))
        store = _mock_store(nl, rank, owners, c, seed=5)
        grp = S.TorchGroup(dist)
        for new_q in (4, 6, 9, 5):
            new = [new_q] + owners[1:] if new_q not in owners else owners
            per = S.exchange_plan(*store, rank, owners, new, c, world)
            got = grp.all_to_all_bytes([S.pack_records(p) for p in per])
            store = S.assemble_store([r for b in got for r in S.unpack_records(b)], nl)
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
