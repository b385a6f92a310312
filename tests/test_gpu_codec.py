"""GPU codec parity: payload bytes, CRC and decoded values bit-identical to
the reference (golden fixture from the reference itself) and to the C oracle.
Reference: codec.cpp:95-266, test_codec.cpp, acceptance.cpp:110-156."""
import hashlib

import numpy as np
import pytest

from golden.inputs import CODEC_CASES, codec_input
from paper_2309_16979_b200 import engine as E

pytestmark = pytest.mark.gpu


def sha(b):
    return hashlib.sha256(b).hexdigest()


def test_golden_codec_cases(engine, golden):
    bad = []
    for case, rec in zip(CODEC_CASES, golden["codec"]):
        amps, forced = codec_input(case)
        payload, crc = engine.compress(amps, case["eb"], forced)
        if len(payload) != rec["len"] or crc != rec["crc"] or sha(payload) != rec["sha256"]:
            bad.append(("enc", case))
            continue
        back = engine.decompress(payload, crc, amps.size)
        if sha(back.tobytes()) != rec["decoded_sha256"]:
            bad.append(("dec", case))
    assert not bad, bad[:5]


def test_known_answer_ones(engine):
    payload, _ = engine.compress(np.ones(4, complex), 0.1)
    assert payload[17:] == bytes([10, 1, 0, 7, 0, 8])


def test_zero_chunk_c16(engine):
    payload, crc = engine.compress(np.zeros(1 << 16, complex), 1e-5)
    assert len(payload) == 2077
    assert (engine.decompress(payload, crc, 1 << 16) == 0).all()


@pytest.mark.parametrize("eb", [0.0, 1e-3, 1e-5, 1e-7, 1e-9])
@pytest.mark.parametrize("c", [1, 4, 8, 12])
def test_batch_matches_oracle(engine, oracle, eb, c):
    rng = np.random.default_rng(c * 100 + int(eb * 1e9))
    n = 1 << c
    count = max(2, 4096 >> c)
    kinds = [rng.uniform(-1, 1, (count, n)) + 1j * rng.uniform(-1, 1, (count, n)),
             (rng.normal(size=(count, n)) + 1j * rng.normal(size=(count, n))) * 2.0 ** -10,
             np.zeros((count, n), complex)]
    for a in kinds:
        a[:, ::7] = 0.0
        got = engine.compress_many(a, eb)
        for k in range(count):
            p, c_ = oracle.compress(a[k], eb)
            assert got[k] == (p, c_), (k, eb, c)
        back = engine.decompress_many([g[0] for g in got], [g[1] for g in got], n)
        for k in range(0, count, max(1, count // 8)):
            ref = oracle.decompress(got[k][0], got[k][1], n)
            assert back[k].tobytes() == ref.tobytes()
        if eb > 0:
            assert np.abs(back.real - a.real).max() <= eb
            assert np.abs(back.imag - a.imag).max() <= eb
        else:
            assert back.tobytes() == np.ascontiguousarray(a).tobytes()


def test_error_bound_mixed_profiles(engine):
    # acceptance.cpp:110-156 style: sparse / uniform / smooth chunks, 3 bounds
    rng = np.random.default_rng(2024)
    for n in (16, 32, 64):
        chunks = []
        for i in range(300):
            v = np.zeros(n, complex)
            if i % 3 == 0:
                v[rng.integers(0, n, 3)] = rng.uniform(-1, 1, 3) + 1j * rng.uniform(-1, 1, 3)
            elif i % 3 == 1:
                v = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
            else:
                t = np.arange(n) / n
                v = np.sin(t + rng.uniform()) + 1j * np.cos(t - rng.uniform()) + 1e-6 * rng.uniform(-1, 1, n)
            chunks.append(v)
        a = np.array(chunks)
        for eb in (1e-3, 1e-5, 1e-7):
            got = engine.compress_many(a, eb)
            back = engine.decompress_many([g[0] for g in got], [g[1] for g in got], n)
            assert np.abs(back.real - a.real).max() <= eb
            assert np.abs(back.imag - a.imag).max() <= eb
        got = engine.compress_many(a, 0.0)
        back = engine.decompress_many([g[0] for g in got], [g[1] for g in got], n)
        assert back.tobytes() == a.tobytes()


def test_flipped_byte_is_caught(engine):
    rng = np.random.default_rng(6)
    a = rng.uniform(-1, 1, 32) + 1j * rng.uniform(-1, 1, 32)
    p, crc = engine.compress(a, 1e-5)
    bad = bytearray(p)
    bad[len(bad) // 2] ^= 0x40
    with pytest.raises(E.CodecError, match="checksum mismatch on chunk 7"):
        engine.decompress(bytes(bad), crc, 32, chunk_index=7)


def test_malformed_payloads(engine, oracle):
    a = np.zeros(8, complex)
    p, _ = oracle.compress(a, 1e-5)
    for mutated in (p[:10], p[:17], p[:-2], p[:17] + bytes([0, 0]) + p[19:]):
        with pytest.raises(E.CodecError, match="malformed|header"):
            engine.decompress(mutated, oracle.crc32(mutated), 8)


def test_invalid_inputs(engine):
    with pytest.raises(E.CodecError):
        engine.compress(np.zeros(3, complex), 1e-5)
    with pytest.raises(E.CodecError):
        engine.compress(np.zeros(4, complex), -1.0)
    with pytest.raises(E.CodecError):
        engine.compress(np.zeros(4, complex), float("nan"))
    with pytest.raises(E.CodecError):
        engine.compress(np.zeros(4, complex), 1e-5, forced=[8])


def test_forced_raws_exact(engine):
    rng = np.random.default_rng(9)
    a = rng.uniform(-1, 1, 16) + 1j * rng.uniform(-1, 1, 16)
    p, crc = engine.compress(a, 1e-2, forced=[0, 16])
    out = engine.decompress(p, crc, 16)
    assert out[0] == a[0]


@pytest.mark.parametrize("eb", [1e-5, 3e-7, 2.0 ** -17, 0.1])
def test_quantiser_half_integer_boundaries(engine, oracle, eb):
    """Values placed on and around the .5 rounding boundaries of the
    quantiser (the division-free fast path must hand these to the exact
    division).  A far value forces a raw reset of the predictor first."""
    rng = np.random.default_rng(int(eb * 1e12) % 2**32)
    far = 40000.0 * 2 * eb
    vals = []
    for k in rng.integers(-32800, 32800, size=1500):
        base = far * (1 if k % 2 else -1)
        step = (float(k) + 0.5) * 2 * eb
        for nudge in (0.0, 1.0, -1.0, 3.0, -3.0):
            v = base + step
            v = np.nextafter(v, np.inf) if nudge > 0 else (np.nextafter(v, -np.inf) if nudge < 0 else v)
            if abs(nudge) == 3.0:
                v = v * (1 + np.sign(nudge) * 2.0 ** -51)
            vals += [0.0, base, float(v)]
    n = 1 << int(np.ceil(np.log2(len(vals))))
    re = np.zeros(n)
    re[: len(vals)] = vals
    amps = re + 1j * np.roll(re, 7)
    got = engine.compress(amps, eb)
    want = oracle.compress(amps, eb)
    assert got == want
    back = engine.decompress(got[0], got[1], n)
    assert back.tobytes() == oracle.decompress(want[0], want[1], n).tobytes()


@pytest.mark.parametrize("eb", [1e-5, 1e-7, 0.01])
def test_fast_forward_tiles_match_oracle(engine, oracle, eb):
    """Tiles that never move the predictor (zero runs, values within 0.99 eb of
    it, -0/+0 mixtures, values straddling the 0.99 eb threshold, forced raws
    inside such runs) take the encoder's and decoder's run fast-forward; the
    bytes must still be the reference's."""
    rng = np.random.default_rng(int(eb * 1e9) + 5)
    n = 1 << 12
    rows = []
    z = np.zeros(n, complex)
    rows.append(z.copy())                                        # all zeros
    a = z.copy(); a[::517] = 0.3 + 0.1j; rows.append(a)          # sparse spikes
    a = np.full(n, 0.25 + 0.0j) + rng.uniform(-0.9, 0.9, n) * eb; rows.append(a)   # smooth
    a = np.full(n, -0.5 + 0.5j); a[1000:1100] += 0.989 * eb; a[2000] += 0.991 * eb
    rows.append(a)                                               # threshold straddle
    a = rng.uniform(-0.98, 0.98, n) * eb + 1j * rng.uniform(-0.98, 0.98, n) * eb
    rows.append(a)                                               # noise below eb
    a = z.copy(); a.real[::3] = -0.0; a.imag[1::5] = -0.0; rows.append(a)   # signed zeros
    a = z.copy(); a[7] = 1.0; a[8] = -1.0; rows.append(a)        # basis-like escapes
    arr = np.array(rows)
    got = engine.compress_many(arr, eb)
    for k in range(len(rows)):
        assert got[k] == oracle.compress(arr[k], eb), k
    back = engine.decompress_many([g[0] for g in got], [g[1] for g in got], n)
    for k in range(len(rows)):
        ref = oracle.decompress(got[k][0], got[k][1], n)
        assert back[k].tobytes() == ref.tobytes(), k
    # forced raws (flat indices) landing inside zero runs
    forced = [5, 64, 4095, n + 33, 2 * n - 1]
    p = engine.compress(z, eb, forced=forced)
    assert p == oracle.compress(z, eb, forced=forced)


@pytest.mark.parametrize("kernel", ["warp", "seg"])
def test_dense_decoders_both_match_golden(golden, tmp_path, kernel):
    """Both dense-store decoders (warp per chunk-half; 8-lane segments, two
    chunks per warp) reproduce the reference's decoded bytes on the golden
    codec corpus and the reference digests of multi-stage lossy runs.
    QZ_DEC_KERNEL is read once per process: fresh subprocess."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    script = (
        "import hashlib, json, sys\n"
        "sys.path.insert(0, 'tests')\n"
        "from golden.inputs import CODEC_CASES, codec_input\n"
        "from paper_2309_16979_b200 import engine as E, circuits as CI\n"
        "from paper_2309_16979_b200.abi import to_array\n"
        "golden = json.load(open('tests/golden/golden.json'))\n"
        "eng = E.Engine()\n"
        "bad = []\n"
        "for case, rec in zip(CODEC_CASES, golden['codec']):\n"
        "    amps, forced = codec_input(case)\n"
        "    if case['eb'] <= 0 or amps.size < 64: continue\n"
        "    p, crc = eng.compress(amps, case['eb'], forced)\n"
        "    back = eng.decompress_many([p] * 3, [crc] * 3, amps.size)\n"
        "    if any(hashlib.sha256(b.tobytes()).hexdigest() != rec['decoded_sha256'] for b in back): bad.append(case)\n"
        "runs = [r for r in golden['runs'] if r['eb'] > 0 and r['stages'] > 1][:4]\n"
        "dig = []\n"
        "for r in runs:\n"
        "    k = r['circuit']\n"
        "    g = CI.qft(int(k.split(':')[1])) if k.startswith('qft:') else CI.ghz(int(k.split(':')[1])) if k.startswith('ghz:') else to_array([(x[0], tuple(x[1]), tuple(x[2])) for x in golden['circuits'][k]])\n"
        "    sim = eng.simulator(r['n'], r['c'], r['m'], r['eb'])\n"
        "    sim.run(g)\n"
        "    dig.append(f'{sim.digest():016x}' == r['digest'])\n"
        "    sim.close()\n"
        "print(json.dumps({'bad': len(bad), 'runs': dig}))\n")
    env = dict(os.environ, QZ_DEC_KERNEL=kernel, PYTHONPATH=str(root))
    res = subprocess.run([sys.executable, "-c", script], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["bad"] == 0 and out["runs"] and all(out["runs"]), out


@pytest.mark.parametrize("kernel", ["staged", "direct"])
def test_encoders_both_match_golden(golden, kernel):
    """Both lossy encoders (pairs staged in shared memory and flushed by
    dedicated warps; each thread writing its own streams) reproduce the
    reference's payload bytes on the golden codec corpus (forced raws
    included) and the reference digests of lossy runs, single- and
    multi-stage.  QZ_ENC_KERNEL is read once per process: fresh subprocess."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    script = (
        "import hashlib, json, sys\n"
        "sys.path.insert(0, 'tests')\n"
        "from golden.inputs import CODEC_CASES, codec_input\n"
        "from paper_2309_16979_b200 import engine as E, circuits as CI\n"
        "from paper_2309_16979_b200.abi import to_array\n"
        "golden = json.load(open('tests/golden/golden.json'))\n"
        "eng = E.Engine()\n"
        "bad = []\n"
        "for case, rec in zip(CODEC_CASES, golden['codec']):\n"
        "    amps, forced = codec_input(case)\n"
        "    if case['eb'] <= 0: continue\n"
        "    p, crc = eng.compress(amps, case['eb'], forced)\n"
        "    if hashlib.sha256(bytes(p)).hexdigest() != rec['sha256'] or crc != rec['crc']: bad.append(case)\n"
        "runs = [r for r in golden['runs'] if r['eb'] > 0][:6]\n"
        "dig = []\n"
        "for r in runs:\n"
        "    k = r['circuit']\n"
        "    g = CI.qft(int(k.split(':')[1])) if k.startswith('qft:') else CI.ghz(int(k.split(':')[1])) if k.startswith('ghz:') else to_array([(x[0], tuple(x[1]), tuple(x[2])) for x in golden['circuits'][k]])\n"
        "    sim = eng.simulator(r['n'], r['c'], r['m'], r['eb'])\n"
        "    sim.run(g)\n"
        "    dig.append(f'{sim.digest():016x}' == r['digest'])\n"
        "    sim.close()\n"
        "print(json.dumps({'bad': len(bad), 'runs': dig}))\n")
    env = dict(os.environ, QZ_ENC_KERNEL=kernel, PYTHONPATH=str(root))
    res = subprocess.run([sys.executable, "-c", script], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["bad"] == 0 and out["runs"] and all(out["runs"]), out
