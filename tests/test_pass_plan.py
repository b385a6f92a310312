"""Host-side fused-pass planning (no GPU): relaxed diagonal units and swap
networks cut the number of HBM sweeps; the strict plan keeps every gate
qubit inside its pass's tile (the replay plan)."""
import pytest

from paper_2309_16979_b200 import circuits as CI
from paper_2309_16979_b200 import engine as E
from tests_util import diagonal_heavy_circuit, random_circuit


def test_qft30_pass_counts():
    g = CI.qft(30)
    rel = E.pass_plan_stats(g, 30, "relaxed")
    strict = E.pass_plan_stats(g, 30, "strict")
    # 27 Hadamard targets above the 3 fixed low bits / 8 free tile bits -> 4
    # passes, the 15-SWAP bit reversal -> 1 permutation pass
    assert rel["passes"] == 5
    assert strict["passes"] > 40
    assert rel["pdiag_ops"] >= 400          # the CP5 runs with a control outside
    assert strict["pdiag_ops"] == 0 and strict["relaxed_groups"] == 0


@pytest.mark.parametrize("name", ["qft", "qaoa", "supremacy", "ghz", "grover"])
def test_relaxed_never_more_passes(name):
    n = 24 if name == "grover" else 28
    g = CI.make(name, n)
    assert (E.pass_plan_stats(g, n, "relaxed")["passes"]
            <= E.pass_plan_stats(g, n, "strict")["passes"])


def test_no_fusion_is_one_pass_per_gate():
    g = random_circuit(16, 40, 3)
    assert E.pass_plan_stats(g, 16, "none")["passes"] == 40


def test_small_buffers_never_relax():
    # a buffer that fits one tile keeps every gate in the tile: nothing to relax
    g = diagonal_heavy_circuit(11, 200, 2)
    st = E.pass_plan_stats(g, 11, "relaxed")
    assert st["relaxed_groups"] == 0 and st["pdiag_ops"] == 0


def test_unsafe_diagonals_relaxed_only_when_checked():
    # Z / S / CZ rows are not +0-safe: the default plan keeps their qubits in
    # the tile; the "checked" plan relaxes them (zero-checked steps, a zero
    # raises the pass's replay flag)
    g = [("h", (q,), ()) for q in range(20)] + [("z", (19,), ()), ("s", (18,), ()),
                                               ("cz", (0, 19), ())]
    assert E.pass_plan_stats(g, 20, "relaxed")["pdiag_ops"] == 0
    assert E.pass_plan_stats(g, 20, "checked")["pdiag_ops"] >= 1
    # supremacy layers: the CZ bricks no longer force their qubits into tiles
    sup = CI.supremacy(30)
    assert E.pass_plan_stats(sup, 30, "checked")["passes"] * 3 < E.pass_plan_stats(sup, 30, "strict")["passes"] * 2


def test_invalid_plan_inputs():
    with pytest.raises(E.QzError):
        E.pass_plan_stats([("h", (20,), ())], 20, "relaxed")
    with pytest.raises(KeyError):
        E.pass_plan_stats([], 20, "bogus")
