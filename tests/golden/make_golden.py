#!/usr/bin/env python3
"""Generate tests/golden/golden.json from the REFERENCE library itself.

Run here (where /root/reference exists and `make -C oracle ref` built
oracle/_ref/libqzref.so):  python tests/golden/make_golden.py

Every expected value in the fixture comes out of the unmodified reference
code (codec.cpp, gates.cpp, kernels.cpp, planner.cpp, pipeline.cpp, store.cpp)
called through oracle/ref_shim.cpp.  Inputs are either stored verbatim or
regenerated from numpy recipes (``inputs.py``) so the fixture stays small.
The GPU box has no /root/reference; tests there compare against this file.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

from oracles import Reference  # noqa: E402
from golden.inputs import CODEC_CASES, KERNEL_CASES, codec_input, kernel_input  # noqa: E402
from paper_2309_16979_b200.abi import from_array, to_array  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def gates_json(arr) -> list:
    return [[name, list(qs), list(ps)] for name, qs, ps in from_array(arr)]


def main() -> None:
    ref = Reference()
    out: dict = {"generator": "tests/golden/make_golden.py", "source": "reference qzsim via oracle/_ref"}

    # ---- gate matrices (gates.cpp:114-182), bit patterns -----------------
    rng = np.random.default_rng(101)
    mats = []
    for name in ["h", "x", "y", "z", "s", "sdg", "t", "tdg", "cx", "cz", "swap"]:
        qs = (0, 1) if name in ("cx", "cz", "swap") else (0,)
        m = ref.gate_matrix((name, qs, ()))
        mats.append({"gate": [name, list(qs), []], "bits": m.view(np.uint64).ravel().tolist()})
    for name, k in [("rx", 1), ("ry", 1), ("rz", 1), ("u1", 1), ("u2", 2), ("u3", 3)]:
        for ps in [[0.0] * k, [-0.0] * k, [np.pi] * k, [-np.pi / 3] * k] + \
                  [list(rng.uniform(-7, 7, k)) for _ in range(12)]:
            ps = [float(p) for p in ps]
            m = ref.gate_matrix((name, (0,), tuple(ps)))
            mats.append({"gate": [name, [0], ps], "bits": m.view(np.uint64).ravel().tolist()})
    out["matrices"] = mats

    # ---- codec (codec.cpp:95-266) ----------------------------------------
    codec = []
    for case in CODEC_CASES:
        amps, forced = codec_input(case)
        payload, crc = ref.compress(amps, case["eb"], forced)
        back = ref.decompress(payload, crc, amps.size)
        rec = dict(case)
        rec.update(len=len(payload), crc=crc, sha256=sha(payload),
                   decoded_sha256=sha(back.tobytes()))
        if len(payload) <= 512:
            rec["payload_hex"] = payload.hex()
        codec.append(rec)
    out["codec"] = codec

    # ---- kernels (kernels.cpp:20-68): buffer + random circuit ------------
    kern = []
    for case in KERNEL_CASES:
        buf = kernel_input(case)
        circ = ref.make_random(case["bits"], case["depth"], case["seed"])
        res = ref.apply_gates(buf, circ)
        kern.append(dict(case, gates=gates_json(circ), sha256=sha(res.tobytes())))
    out["kernels"] = kern

    # ---- circuits + planner + full runs ----------------------------------
    runs = []
    small = []
    for seed in range(1, 41):
        n = 4 + seed % 9
        circ = ref.make_random(n, 60, seed)
        for c in (2, 4):
            for m in (c + 2, c + 4):
                if m > n:
                    continue
                for eb in (0.0, 1e-3, 1e-5, 1e-7):
                    if (seed + c + m) % 4 != int(eb and -np.log10(eb)) % 4 and eb != 1e-5:
                        continue
                    r = ref.run(n, circ, c, m, eb, workers=2)
                    small.append(dict(n=n, c=c, m=m, eb=eb, circuit=f"random:{n}:60:{seed}",
                                      digest=f"{r['digest']:016x}", norm=r["norm"],
                                      stages=r["stages"], current_bytes=r["current_bytes"],
                                      peak_bytes=r["peak_bytes"]))
    circuits = {}
    for seed in range(1, 41):
        n = 4 + seed % 9
        circuits[f"random:{n}:60:{seed}"] = gates_json(ref.make_random(n, 60, seed))
    # SURVEY §8(c) digests plus a few more families
    big = [("random", 12, 80, 8, 4, 8, 1e-5), ("qft", 20, 0, 0, 16, 20, 1e-5),
           ("qft", 20, 0, 0, 12, 16, 1e-5), ("ghz", 20, 0, 0, 16, 20, 1e-5),
           ("qft", 20, 0, 0, 16, 20, 0.0), ("random", 20, 200, 1, 16, 20, 1e-5),
           ("ghz", 24, 0, 0, 16, 20, 1e-5), ("random", 24, 200, 1, 16, 20, 1e-7),
           ("qft", 16, 0, 0, 8, 12, 1e-7), ("ghz", 16, 0, 0, 8, 12, 1e-6),
           ("random", 14, 40, 14, 8, 12, 1e-6), ("qft", 18, 0, 0, 12, 16, 1e-5),
           ("random", 18, 60, 9, 12, 16, 1e-5), ("qft", 22, 0, 0, 14, 22, 1e-5),
           ("ghz", 26, 0, 0, 16, 22, 1e-5)]
    for fam, n, depth, seed, c, m, eb in big:
        if fam == "random":
            circ = ref.make_random(n, depth, seed)
            key = f"random:{n}:{depth}:{seed}"
            circuits[key] = gates_json(circ)
        elif fam == "qft":
            circ, key = ref.make_qft(n), f"qft:{n}"
        else:
            circ, key = ref.make_ghz(n), f"ghz:{n}"
        t = time.time()
        r = ref.run(n, circ, c, m, eb, workers=0)
        runs.append(dict(n=n, c=c, m=m, eb=eb, circuit=key, digest=f"{r['digest']:016x}",
                         norm=r["norm"], stages=r["stages"], current_bytes=r["current_bytes"],
                         peak_bytes=r["peak_bytes"], ratio=r["ratio"],
                         total_payload=r["total_payload"], ref_wall_seconds=r["wall_seconds"]))
        print(f"{key} c={c} m={m} eb={eb}: {r['digest']:016x} stages={r['stages']} "
              f"{time.time() - t:.1f}s", flush=True)
    out["circuits"] = circuits
    out["runs_small"] = small
    out["runs"] = runs

    plans = []
    for seed in range(1, 21):
        n = 4 + seed % 8
        circ = ref.make_random(n, 50, seed)
        for c in (1, 2, 3):
            for m in range(c + 2, n + 1):
                plans.append(dict(circuit=f"random:{n}:50:{seed}", n=n, c=c, m=m,
                                  stages=[[g, h] for g, h in ref.plan(n, circ, c, m)]))
        circuits[f"random:{n}:50:{seed}"] = gates_json(circ)
    out["plans"] = plans
    qft = {str(n): gates_json(ref.make_qft(n)) for n in (3, 5, 8)}
    out["generators"] = {"qft": qft, "ghz": {str(n): gates_json(ref.make_ghz(n)) for n in (3, 6)}}

    (HERE / "golden.json").write_text(json.dumps(out, separators=(",", ":")))
    print("wrote", HERE / "golden.json", (HERE / "golden.json").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
