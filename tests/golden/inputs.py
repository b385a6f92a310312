"""Deterministic input recipes for the golden fixtures (numpy PCG64 streams).

make_golden.py feeds these inputs to the reference; the tests regenerate the
same inputs and compare the engine's bytes with the recorded expectations.
"""
from __future__ import annotations

import numpy as np

__all__ = ["CODEC_CASES", "KERNEL_CASES", "codec_input", "kernel_input"]


def _cases() -> list[dict]:
    cases = [dict(kind="ones", n=4, eb=0.1, seed=0)]  # test_codec.cpp:74-98
    for n in (1, 2, 64, 1 << 16):
        for eb in (1e-5, 0.0):
            cases.append(dict(kind="zeros", n=n, eb=eb, seed=0))
    seed = 1
    for n in (1, 2, 16, 128, 1024, 4096):
        for eb in (1e-3, 1e-5, 1e-7, 0.0):
            cases.append(dict(kind="uniform", n=n, eb=eb, seed=seed))
            seed += 1
    for n in (256, 4096, 16384):
        for eb in (1e-7, 1e-8, 1e-9):
            cases.append(dict(kind="gauss", n=n, eb=eb, seed=seed, sigma_log2=-10.5))
            seed += 1
    for n in (16, 32, 64, 512):
        for kind in ("sparse", "smooth", "ghzlike", "boundary", "ties", "edge", "special"):
            for eb in (1e-3, 1e-5, 1e-7, 0.0):
                cases.append(dict(kind=kind, n=n, eb=eb, seed=seed))
                seed += 1
    for n in (64, 4096):
        cases.append(dict(kind="boundary_long", n=n, eb=1e-5, seed=seed))
        seed += 1
        cases.append(dict(kind="bits", n=n, eb=0.0, seed=seed))
        seed += 1
    for n in (16, 256):
        for eb in (1e-2, 1e-5):
            cases.append(dict(kind="forced", n=n, eb=eb, seed=seed))
            seed += 1
    return cases


CODEC_CASES = _cases()


def _pack(v: np.ndarray, n: int) -> np.ndarray:
    """Interleave planes without complex arithmetic (keeps inf/NaN/-0 bits)."""
    raw = np.empty(2 * n, dtype=np.float64)
    raw[0::2], raw[1::2] = v[:n], v[n:]
    return raw.view(np.complex128)


def codec_input(case: dict) -> tuple[np.ndarray, list[int]]:
    n, kind = case["n"], case["kind"]
    rng = np.random.default_rng(case["seed"])
    forced: list[int] = []
    a = np.zeros(n, dtype=np.complex128)
    if kind == "ones":
        a[:] = 1.0
    elif kind == "zeros":
        pass
    elif kind == "uniform":
        a = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    elif kind == "gauss":
        s = 2.0 ** case["sigma_log2"]
        a = rng.normal(0, s, n) + 1j * rng.normal(0, s, n)
    elif kind == "sparse":  # acceptance.cpp:121-124
        for _ in range(3):
            a[rng.integers(0, n)] = complex(rng.uniform(-1, 1), rng.uniform(-1, 1))
    elif kind == "smooth":  # acceptance.cpp:128-134
        ph, fr = rng.uniform(-1, 1), 2 * rng.uniform(-1, 1)
        t = np.arange(n) / n
        a = (np.sin(fr * t + ph) + 1e-6 * rng.uniform(-1, 1, n)) + \
            1j * (np.cos(fr * t - ph) + 1e-6 * rng.uniform(-1, 1, n))
    elif kind == "ghzlike":
        r = 0.7071067811865476
        a[0] = r
        a[rng.integers(1, n)] = -r
        a[n - 1] = complex(-0.0, -0.0)
        a[n // 2] = complex(0.0, -0.0)
    elif kind == "boundary":
        # runs that straddle the real→imag plane boundary of the byte planes
        re = np.zeros(n)
        im = np.zeros(n)
        re[: rng.integers(1, n)] = 0.25
        im[rng.integers(0, n):] = 0.5
        a = re + 1j * im
    elif kind == "boundary_long":
        re = np.zeros(n)
        im = np.zeros(n)
        re[n - 1 - int(rng.integers(0, 300)) % n] = 0.125
        im[int(rng.integers(0, 300)) % n] = 0.375
        a = re + 1j * im
    elif kind == "ties":
        eb = case["eb"] or 2.0 ** -10
        k = rng.integers(-40000, 40000, size=2 * n)
        v = (k.astype(np.float64)) * eb  # odd k → exact .5 quotients
        a = _pack(v, n)
    elif kind == "edge":
        eb = case["eb"] or 1e-5
        d = rng.integers(-4, 5, size=2 * n).astype(np.float64)
        v = (32767.5 + d * 1e-12) * 2 * eb * rng.choice([-1.0, 1.0], size=2 * n)
        v[::3] = 0.0  # reset the predictor often so the edge stays in reach
        a = _pack(v, n)
    elif kind == "special":
        pool = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, 5e-324, -2.2e-308, 1e308,
                         -1e308, 1.0, -1.0, 0.5, 1e-20])
        v = pool[rng.integers(0, pool.size, size=2 * n)]
        a = _pack(v, n)
    elif kind == "bits":
        # exact bit patterns, NaN payloads included
        v = rng.integers(0, 2**63, size=2 * n, dtype=np.uint64).view(np.float64)
        raw = np.empty(2 * n, dtype=np.float64)
        raw[0::2], raw[1::2] = v[:n], v[n:]
        a = raw.view(np.complex128)
    elif kind == "forced":
        a = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        forced = sorted(set([0, n] + [int(x) for x in rng.integers(0, 2 * n, size=5)]))
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(a, dtype=np.complex128), forced


KERNEL_CASES = [dict(bits=b, depth=d, seed=s) for b, d, s in
                [(1, 10, 1), (2, 20, 2), (3, 40, 3), (5, 60, 4), (8, 80, 5), (10, 120, 6),
                 (12, 200, 7), (14, 100, 8)]]


def kernel_input(case: dict) -> np.ndarray:
    rng = np.random.default_rng(1000 + case["seed"])
    n = 1 << case["bits"]
    a = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    a[rng.integers(0, n, size=max(1, n // 8))] = 0.0  # exact zeros exercise ±0 rules
    return np.ascontiguousarray(a)
