"""GPU pipeline parity: final store digest, footprint and stage counts equal
to the reference's run() on the same circuit (golden fixture produced by the
reference).  Mirrors test_pipeline.cpp and acceptance.cpp C1/C4/C5/C8."""
import numpy as np
import pytest

from paper_2309_16979_b200 import engine as E
from paper_2309_16979_b200.abi import to_array

pytestmark = pytest.mark.gpu


def circuit(golden, oracle, key):
    if key.startswith("qft:"):
        return oracle.make_qft(int(key.split(":")[1]))
    if key.startswith("ghz:"):
        return oracle.make_ghz(int(key.split(":")[1]))
    return to_array([(g[0], tuple(g[1]), tuple(g[2])) for g in golden["circuits"][key]])


def run_sim(engine, n, c, m, eb, gates, **kw):
    sim = engine.simulator(n, c, m, eb, **kw)
    sim.run(gates)
    return sim


def test_small_runs_digest(engine, oracle, golden):
    bad = []
    for rec in golden["runs_small"]:
        g = circuit(golden, oracle, rec["circuit"])
        sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g)
        st = sim.stats()
        if (f"{sim.digest():016x}" != rec["digest"] or st["stages"] != rec["stages"]
                or st["current_bytes"] != rec["current_bytes"]):
            bad.append(rec)
        sim.close()
    assert not bad, bad[:3]


@pytest.mark.parametrize("idx", range(15))
def test_large_runs_digest(engine, oracle, golden, idx):
    rec = golden["runs"][idx]
    g = circuit(golden, oracle, rec["circuit"])
    sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g)
    assert f"{sim.digest():016x}" == rec["digest"], rec
    st = sim.stats()
    assert st["stages"] == rec["stages"]
    assert st["current_bytes"] == rec["current_bytes"]
    assert sim.payload_bytes() == rec["total_payload"]
    assert sim.norm() == pytest.approx(rec["norm"], abs=1e-9)


def test_small_window_same_digest(engine, oracle, golden):
    # scheduling knobs (window size, fusion) never change the bytes
    rec = golden["runs"][0]
    g = circuit(golden, oracle, rec["circuit"])
    for window in (1 << rec["m"], 1 << (rec["m"] + 1), 0):
        for fuse in (True, False):
            sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g,
                          window_amps=window, fuse=fuse)
            assert f"{sim.digest():016x}" == rec["digest"]


def test_empty_circuit_is_init(engine, oracle):
    sim = engine.simulator(6, 2, 4, 0.0)
    d0 = sim.digest()
    sim.run([])
    assert sim.digest() == d0
    assert sim.norm() == 1.0
    r = oracle.run(6, [], 2, 4, 0.0)
    assert r["digest"] == d0


def test_init_basis_exact(engine):
    for eb in (0.0, 1e-3, 1e-5, 0.3):
        sim = engine.simulator(6, 3, 5, eb)
        s = sim.state()
        assert abs(s[0] - 1) <= 1e-12 and (s[1:] == 0).all()
        assert sim.norm() == 1.0


def test_init_ratios(engine):
    assert engine.simulator(20, 12, 16, 1e-5).stats()["ratio"] > 100
    st = engine.simulator(24, 16, 20, 1e-5).stats()
    assert st["current_bytes"] * 100 <= st["dense_bytes"]


def test_lossless_matches_dense(engine, oracle):
    g = to_array([])
    rng = np.random.default_rng(77)
    from tests_util import random_circuit
    g = random_circuit(10, 50, 77)
    dense = oracle.dense(10, g)
    for c, m in ((4, 6), (2, 4), (3, 8)):
        sim = run_sim(engine, 10, c, m, 0.0, g)
        assert np.abs(sim.state() - dense).max() <= 1e-12


def test_fidelity_vs_gpu_dense(engine, oracle):
    g = oracle.make_ghz(16)
    sim = run_sim(engine, 16, 8, 12, 1e-6, g)
    dense = engine.dense_state(16, g)
    assert sim.fidelity(dense) >= 0.9999
    ref = oracle.dense(16, g)
    assert abs(sim.fidelity(dense) - oracle.fidelity(ref, sim.state())) < 1e-12


def test_export_import_roundtrip(engine, oracle, golden):
    rec = golden["runs"][0]
    g = circuit(golden, oracle, rec["circuit"])
    sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g)
    blob, sizes, crcs = sim.export()
    other = engine.simulator(rec["n"], rec["c"], rec["m"], rec["eb"], init=False)
    other.import_(blob, sizes, crcs)
    assert other.digest() == sim.digest()
    ref = oracle.run(rec["n"], g, rec["c"], rec["m"], rec["eb"], export=True)
    assert ref["payload"] == blob


def test_write_and_read_chunk(engine, oracle):
    rng = np.random.default_rng(21)
    sim = engine.simulator(8, 4, 6, 1e-4)
    before = sim.stats()["current_bytes"]
    vals = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    sim.write_chunk(5, vals)
    back = sim.read_chunks(5, 1)
    assert np.abs(back.real - vals.real).max() <= 1e-4
    assert np.abs(back.imag - vals.imag).max() <= 1e-4
    old = len(oracle.compress(np.zeros(16, complex), 1e-4)[0])
    new = len(oracle.compress(vals, 1e-4)[0])
    assert sim.stats()["current_bytes"] == before - old + new
    with pytest.raises(E.StoreError):
        sim.read_chunks(16, 1)


def test_invalid_configs(engine):
    with pytest.raises(E.StoreError):
        engine.simulator(10, 12, 14, 0.0)
    with pytest.raises(E.StoreError):
        engine.simulator(41, 16, 20, 0.0)
    with pytest.raises(E.PlanError):
        engine.simulator(6, 4, 4, 0.0).run([("h", (0,), ())])      # m - c < 2
    with pytest.raises(E.PlanError):
        engine.simulator(6, 2, 6, 0.0).run([("h", (7,), ())])      # bad qubit


@pytest.mark.parametrize("idx", [0, 1, 2, 5, 7, 9])
def test_host_staged_same_digest(engine, oracle, golden, idx):
    """Compressed store in mapped page-locked host memory, streamed through
    HBM windows: same payload bytes as the HBM-resident run and the reference."""
    rec = golden["runs"][idx]
    g = circuit(golden, oracle, rec["circuit"])
    sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g, residency="host")
    assert f"{sim.digest():016x}" == rec["digest"], rec
    st = sim.stats()
    assert st["current_bytes"] == rec["current_bytes"]
    assert st["h2d_bytes"] > 0 and st["d2h_bytes"] > 0


def test_host_staged_windows_and_io(engine, oracle, golden):
    rec = golden["runs"][0]
    g = circuit(golden, oracle, rec["circuit"])
    for window in (1 << rec["m"], 1 << (rec["m"] + 1)):
        sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g, residency="host",
                      window_amps=window)
        assert f"{sim.digest():016x}" == rec["digest"]
        blob, sizes, crcs = sim.export()
        assert oracle.fnv1a64(blob) == sim.digest()


@pytest.mark.parametrize("key,g", [(("random:12:80:8", 4, 8, 1e-5), 1), (("random:12:80:8", 4, 8, 1e-5), 2),
                                   (("qft:20", 12, 16, 1e-5), 2), (("qft:20", 12, 16, 1e-5), 1),
                                   (("random:24:200:1", 16, 20, 1e-7), 2)])
def test_sharded_ranks_same_digest(engine, oracle, golden, key, g):
    """2^g ranks (in-process, one GPU) exchanging compressed chunks at stage
    boundaries reproduce the single-GPU / reference digest."""
    from paper_2309_16979_b200 import sharding as S
    circ_key, c, m, eb = key
    rec = next(r for r in golden["runs"] if r["circuit"] == circ_key and r["c"] == c
               and r["m"] == m and r["eb"] == eb)
    gl = circuit(golden, oracle, circ_key)
    run = S.ShardedRun(engine, rec["n"], c, m, eb, g, range(1 << g), S.LocalGroup(1 << g))
    run.init_basis()
    run.run(gl)
    assert f"{run.digest():016x}" == rec["digest"]


def _relax_cases():
    from paper_2309_16979_b200 import circuits as CI
    from tests_util import diagonal_heavy_circuit
    return [
        ("qft16", 16, 8, 16, 1e-5, lambda: CI.qft(16)),
        ("qft18_m14", 18, 8, 14, 1e-5, lambda: CI.qft(18)),
        ("qaoa16", 16, 8, 16, 1e-5, lambda: CI.qaoa(16)),
        ("supremacy16", 16, 8, 16, 1e-6, lambda: CI.supremacy(16, depth=8)),
        ("ghz16_phases", 16, 8, 16, 0.0,
         lambda: to_array([(g[0], g[1], g[2]) for g in
                           [("h", (0,), ())] + [("cx", (0, k), ()) for k in range(1, 16)]
                           + [("z", (15,), ()), ("s", (14,), ()), ("cz", (3, 12), ()),
                              ("u1", (13,), (0.3,)), ("h", (15,), ()), ("cz", (15, 2), ())]])),
        ("diag_heavy_a", 16, 8, 16, 0.0, lambda: to_array(diagonal_heavy_circuit(16, 300, 5))),
        ("diag_heavy_b", 16, 6, 14, 1e-6, lambda: to_array(diagonal_heavy_circuit(16, 400, 9))),
    ]


@pytest.mark.parametrize("case", range(7))
def test_relaxed_passes_match_strict_and_reference(engine, oracle, case):
    """Diagonal units with qubits outside the pass's tile set (relaxed plan),
    the strict plan, and a forced device-side replay all give the reference's
    bytes (oracle digest)."""
    name, n, c, m, eb, make = _relax_cases()[case]
    g = make()
    ref = oracle.run(n, g, c, m, eb)["digest"]
    out = {}
    for mode, kw in (("relaxed", {}), ("strict", {"fuse": "strict"}),
                     ("replay", {"force_replay": True}), ("checked", {"fuse": "checked"}),
                     ("checked_replay", {"fuse": "checked", "force_replay": True})):
        sim = run_sim(engine, n, c, m, eb, g, **kw)
        out[mode] = (sim.digest(), sim.stats())
        sim.close()
    for mode, (d, _) in out.items():
        assert d == ref, (name, mode)
    rel, strict, rep = out["relaxed"][1], out["strict"][1], out["replay"][1]
    assert rel["gate_passes"] <= strict["gate_passes"], name
    assert strict["replays"] == 0
    if rel["gate_passes"] < strict["gate_passes"]:
        assert rep["replays"] >= 1, name


def test_relaxed_qft_needs_no_replay(engine):
    from paper_2309_16979_b200 import circuits as CI
    sim = run_sim(engine, 20, 10, 20, 1e-5, CI.qft(20))
    st = sim.stats()
    assert st["replays"] == 0
    strict = run_sim(engine, 20, 10, 20, 1e-5, CI.qft(20), fuse="strict")
    assert strict.digest() == sim.digest()
    assert st["gate_passes"] * 3 < strict.stats()["gate_passes"]


def _load_state(engine, oracle, n, c, m, state):
    """Lossless store holding `state` exactly (payloads from the oracle codec)."""
    sim = engine.simulator(n, c, m, 0.0, init=False)
    blobs, sizes, crcs = [], [], []
    for k in range(1 << (n - c)):
        p, crc = oracle.compress(state[k << c:(k + 1) << c], 0.0)
        blobs.append(p)
        sizes.append(len(p))
        crcs.append(crc)
    sim.import_(b"".join(blobs), np.array(sizes, np.uint32), np.array(crcs, np.uint32))
    return sim


def _random_state(rng, n, neg_zero: bool):
    st = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)) / (1 << (n // 2))
    st[rng.random(1 << n) < 0.1] = 0.0                         # +0 components
    if neg_zero:
        z = rng.random(1 << n) < 0.02
        st.real[z] = -0.0
    return st


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("neg_zero", [False, True])
def test_swap_network_pass_bit_exact(engine, oracle, seed, neg_zero):
    """Runs of disjoint SWAPs become one in-place bit-permutation pass; the
    result equals the reference kernels bit for bit, and a -0 component makes
    the pass replay strictly (still bit-exact)."""
    rng = np.random.default_rng(100 + seed)
    n, c = 14, 4
    q = rng.permutation(n)
    npairs = int(rng.integers(2, n // 2 + 1))
    gates = [("swap", (int(q[2 * i]), int(q[2 * i + 1])), ()) for i in range(npairs)]
    if seed % 2:
        gates = [("h", (int(q[0]),), ()), ("t", (int(q[1]),), ())] + gates + [("rx", (3,), (0.4,))]
    state = _random_state(rng, n, neg_zero)
    want = oracle.apply_gates(state.copy(), gates)
    sim = _load_state(engine, oracle, n, c, n, state)
    sim.run(gates)
    got = sim.state()
    assert got.view(np.uint64).tobytes() == want.view(np.uint64).tobytes()
    if neg_zero:
        assert sim.stats()["replays"] >= 1
    elif seed % 2 == 0:
        assert sim.stats()["replays"] == 0


def test_export_into_pinned_buffer(engine, oracle, golden):
    rec = golden["runs"][0]
    g = circuit(golden, oracle, rec["circuit"])
    sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g)
    blob, sizes, crcs = sim.export()
    out = engine.pinned(len(blob) + 100)
    view, s2, c2 = sim.export(out, engine.pinned(4 * sim.chunk_count, np.uint32),
                              engine.pinned(4 * sim.chunk_count, np.uint32))
    assert view.tobytes() == blob and (s2 == sizes).all() and (c2 == crcs).all()
    with pytest.raises(ValueError):
        sim.export(engine.pinned(8))


@pytest.mark.parametrize("seed", range(10))
def test_random_circuits_relaxed_vs_reference(engine, oracle, seed):
    """Seeded random circuits over the whole gate set plus diagonal-unit runs,
    windows wider than one tile (relaxed passes, swap networks, replays):
    final store digest equals the reference's."""
    from tests_util import diagonal_heavy_circuit, random_circuit
    rng = np.random.default_rng(1000 + seed)
    n = 14
    g = random_circuit(n, 60, 2000 + seed) + diagonal_heavy_circuit(n, 80, 3000 + seed)
    q = rng.permutation(n)
    g += [("swap", (int(q[2 * i]), int(q[2 * i + 1])), ()) for i in range(int(rng.integers(2, 6)))]
    g += random_circuit(n, 20, 4000 + seed)
    eb = [0.0, 1e-7, 1e-5][seed % 3]
    c, m = (4, 14) if seed % 2 else (6, 12)
    ref = oracle.run(n, g, c, m, eb)["digest"]
    for fuse in (True, "checked"):
        sim = run_sim(engine, n, c, m, eb, g, fuse=fuse)
        assert sim.digest() == ref, fuse
        sim.close()


def test_qft30_full_size_parity(engine, oracle):
    """Beyond the oracle's reach: at the bench size the relaxed
    plan (< 16 passes) and the strict plan (54 passes) give the same store bytes,
    and sampled chunks decode through the C oracle to the GPU's values."""
    from paper_2309_16979_b200 import circuits as CI
    g = CI.qft(30)
    sim = run_sim(engine, 30, 16, 30, 1e-5, g)
    d_rel = sim.digest()
    blob, sizes, crcs = sim.export()
    offs = np.concatenate([[0], np.cumsum(sizes.astype(np.int64))])
    rng = np.random.default_rng(30)
    for k in [0, 1, sim.chunk_count - 1] + list(rng.integers(0, sim.chunk_count, 5)):
        k = int(k)
        p = blob[offs[k]:offs[k + 1]]
        assert oracle.crc32(p) == int(crcs[k])
        want = oracle.decompress(p, int(crcs[k]), 1 << 16)
        got = sim.read_chunks(k, 1)
        assert got.tobytes() == want.tobytes(), k
    # a handful of tile passes + the swap network (the fresh-qubit planning
    # splits the |0>-heavy start into passes over dense live tiles)
    assert sim.stats()["gate_passes"] < 16
    sim.close()
    strict = run_sim(engine, 30, 16, 30, 1e-5, g, fuse="strict")
    assert strict.digest() == d_rel
    strict.close()
    # the bench config's digest, generated by the unmodified reference
    # (tests/golden/make_golden_r2.py); pinned once the fixture holds it
    rec = [r for r in _r2_cases() if (r["circuit"], r["n"], r["m"]) == ("qft", 30, 30)]
    if rec:
        assert f"{d_rel:016x}" == rec[0]["digest"]


def _r2_cases():
    import json
    from pathlib import Path
    f = Path(__file__).parent / "golden" / "golden_r2.json"
    return json.loads(f.read_text()) if f.exists() else []


@pytest.mark.parametrize("idx", range(9))
def test_baseline_configs_vs_reference(engine, idx):
    """BASELINE.json's own configs against digests of the unmodified
    reference (tests/golden/make_golden_r2.py): QFT-30 / GHZ-30 at the bench
    config (c=16 m=30 eb=1e-5), multi-stage QFT-30 (m=26) and GHZ-30 (m=20),
    and the Grover / QAOA families (cfg4) — digest, stage count and store
    bytes equal."""
    from paper_2309_16979_b200 import circuits as CI
    cases = _r2_cases()
    if idx >= len(cases):
        pytest.skip("golden_r2.json case not generated yet")
    rec = cases[idx]
    g = CI.make(rec["circuit"], rec["n"], **rec["kw"])
    assert len(g) == rec["gates"]
    sim = run_sim(engine, rec["n"], rec["c"], rec["m"], rec["eb"], g)
    st = sim.stats()
    assert f"{sim.digest():016x}" == rec["digest"], rec
    assert st["stages"] == rec["stages"]
    assert st["current_bytes"] == rec["current_bytes"]
    sim.close()


def _large_cases():
    import json
    from pathlib import Path
    f = Path(__file__).parent / "golden" / "golden_large.json"
    return json.loads(f.read_text()) if f.exists() else []


@pytest.mark.parametrize("idx", range(4))
def test_large_runs_vs_reference(engine, idx):
    """Reference digests at 2^26..2^28 (tests/golden/make_golden_large.py):
    relaxed passes, swap networks and multi-stage windows at scale."""
    from paper_2309_16979_b200 import circuits as CI
    cases = _large_cases()
    if idx >= len(cases):
        pytest.skip("golden_large.json not generated")
    rec = cases[idx]
    n = rec["n"]
    g = CI.supremacy(n, **rec["kw"]) if rec["circuit"] == "supremacy" else CI.make(rec["circuit"], n)
    sim = run_sim(engine, n, rec["c"], rec["m"], rec["eb"], g)
    st = sim.stats()
    assert f"{sim.digest():016x}" == rec["digest"], rec
    assert st["stages"] == rec["stages"]
    assert st["current_bytes"] == rec["current_bytes"]
    sim.close()


@pytest.mark.parametrize("fuse,force", [(True, True), ("checked", False), ("checked", True)])
def test_host_staged_replay_modes(engine, oracle, fuse, force):
    """Host-staged pipeline (gather / compute / write-back streams) with the
    window-level and the per-pass replays forced or taken: reference bytes."""
    from tests_util import diagonal_heavy_circuit
    n, c, m, eb = 15, 6, 14, 1e-6
    g = to_array(diagonal_heavy_circuit(n, 200, 77))
    ref = oracle.run(n, g, c, m, eb)["digest"]
    sim = run_sim(engine, n, c, m, eb, g, residency="host", fuse=fuse, force_replay=force)
    assert sim.digest() == ref
    if force:
        assert sim.stats()["replays"] >= 1



def test_full_case_set_same_digest(engine, golden, oracle, tmp_path):
    """The per-pass case-set choice (tile_pass_reg<kPassDiagH / kPassGen>) only
    changes speed: with QZ_NO_NARROW=1 (every pass on the full jump table) the
    reference-generated digests hold too.  Fresh process: the switch is read
    once per process."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    recs = [r for r in golden["runs"] if r["circuit"].startswith(("qft:", "ghz:"))][:3]
    recs += [r for r in golden["runs"] if not r["circuit"].startswith(("qft:", "ghz:"))][:2]
    for i, rec in enumerate(recs):
        np.save(tmp_path / f"g{i}.npy", circuit(golden, oracle, rec["circuit"]))
    script = (
        "import json, sys\n"
        "import numpy as np\n"
        "from paper_2309_16979_b200 import engine as E\n"
        "recs, d = json.loads(sys.argv[1]), sys.argv[2]\n"
        "eng = E.Engine()\n"
        "out = []\n"
        "for i, rec in enumerate(recs):\n"
        "    sim = eng.simulator(rec['n'], rec['c'], rec['m'], rec['eb'])\n"
        "    sim.run(np.load(f'{d}/g{i}.npy'))\n"
        "    out.append(f'{sim.digest():016x}')\n"
        "    sim.close()\n"
        "print(json.dumps(out))\n")
    env = dict(os.environ, QZ_NO_NARROW="1", PYTHONPATH=str(root))
    res = subprocess.run([sys.executable, "-c", script, json.dumps(recs), str(tmp_path)],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert json.loads(res.stdout.strip().splitlines()[-1]) == [r["digest"] for r in recs]


@pytest.mark.parametrize("switch,kw", [("QZ_NO_NZMAP", {}), ("QZ_NO_NZMAP", {"fuse": "checked"}),
                                    ("QZ_NO_NZMAP", {"force_replay": True}),
                                    ("QZ_NO_NZMAP", {"residency": "host"}),
                                    ("QZ_NO_WMAP", {}), ("QZ_NO_WMAP", {"fuse": "checked"}),
                                    ("QZ_NO_FRESH", {}), ("QZ_NO_FRESH", {"fuse": "checked"}),
                                    ("QZ_NO_FRESH", {"residency": "host"}),
                                    ("QZ_NO_PERM_FUSE", {}), ("QZ_NO_PERM_FUSE", {"force_replay": True}),
                                    ("QZ_NO_ABSORB", {}), ("QZ_NO_ABSORB", {"force_replay": True}),
                                    ("QZ_NO_DIRECT", {}), ("QZ_NO_DIRECT", {"fuse": "checked"})])
def test_skip_switches_off_same_digest(engine, golden, oracle, tmp_path, switch, kw):
    """Work-skipping devices only skip work: with QZ_NO_NZMAP=1 (no tile
    skipped on the zero-slot map's say-so), QZ_NO_WMAP=1 (register groups
    on the plain thread map, no warp-uniform block skips), QZ_NO_FRESH=1 (no
    fresh-qubit planning, dead-chunk skipping or static +0 registers),
    QZ_NO_PERM_FUSE=1 (swap networks as their own pass) or QZ_NO_ABSORB=1
    (no trailing swap network absorbed into the stage layout) or QZ_NO_DIRECT=1
    (single-group passes through the shared-memory tile) the reference
    digests hold for the relaxed, checked, forced-replay and host-staged
    variants.  Fresh process: the switches are read once per process."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    recs = [r for r in golden["runs"] if r["circuit"].startswith(("qft:", "ghz:"))][:3]
    recs += [r for r in golden["runs"] if not r["circuit"].startswith(("qft:", "ghz:"))][:2]
    for i, rec in enumerate(recs):
        np.save(tmp_path / f"g{i}.npy", circuit(golden, oracle, rec["circuit"]))
    script = (
        "import json, sys\n"
        "import numpy as np\n"
        "from paper_2309_16979_b200 import engine as E\n"
        "recs, d, kw = json.loads(sys.argv[1]), sys.argv[2], json.loads(sys.argv[3])\n"
        "eng = E.Engine()\n"
        "out = []\n"
        "for i, rec in enumerate(recs):\n"
        "    sim = eng.simulator(rec['n'], rec['c'], rec['m'], rec['eb'], **kw)\n"
        "    sim.run(np.load(f'{d}/g{i}.npy'))\n"
        "    out.append(f'{sim.digest():016x}')\n"
        "    sim.close()\n"
        "print(json.dumps(out))\n")
    env = dict(os.environ, PYTHONPATH=str(root))
    env[switch] = "1"
    res = subprocess.run([sys.executable, "-c", script, json.dumps(recs), str(tmp_path),
                          json.dumps(kw)], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert json.loads(res.stdout.strip().splitlines()[-1]) == [r["digest"] for r in recs]


@pytest.mark.parametrize("eb", [1e-5, 0.0])
def test_repeated_init_same_bytes(engine, oracle, eb):
    """init_basis on a simulator that was already initialised copies the
    first init's payloads back (no codec round trip): every later run from
    it reproduces the oracle's store bytes, single- and multi-stage."""
    from paper_2309_16979_b200 import circuits as CI
    for n, c, m in ((14, 8, 14), (14, 8, 11)):
        g = CI.qft(n)
        want = oracle.run(n, g, c, m, eb)["digest"]
        sim = engine.simulator(n, c, m, eb, init=False)
        try:
            for _ in range(3):
                sim.init_basis()
                sim.run(g)
                assert sim.digest() == want, (n, c, m, eb)
        finally:
            sim.close()
