"""The engine's stage planner (qzc_plan_export: csrc/qz_plan.cu, host code in
libqzcuda.so, no GPU needed) against the 258 plans the UNMODIFIED reference
produced (tests/golden/make_golden.py: qzsim::plan over 20 random circuits x
c in {1,2,3} x every m; planner.cpp:46-96 greedy split, 32-42 padding).
Also the C++ drop-in's plan() (libqzsim_b200.so) through the same fixture."""
import ctypes as C

import numpy as np
import pytest

from paper_2309_16979_b200 import engine
from paper_2309_16979_b200.abi import to_array
from paper_2309_16979_b200.sharding import global_stages


def _circ(golden, key):
    return to_array([(g[0], tuple(g[1]), tuple(g[2])) for g in golden["circuits"][key]])


def test_fixture_has_all_plans(golden):
    assert len(golden["plans"]) == 258


def test_engine_planner_matches_reference_plans(golden):
    bad = []
    for rec in golden["plans"]:
        g = _circ(golden, rec["circuit"])
        got = global_stages(rec["n"], rec["c"], rec["m"], g)
        want = rec["stages"]
        got_l = [[s.count, s.high] for s in got]
        if got_l != want:
            bad.append((rec["circuit"], rec["c"], rec["m"]))
        # stages tile the gate list in order
        assert [s.first for s in got] == list(np.cumsum([0] + [s.count for s in got])[:-1])
    assert not bad, bad[:5]


def test_planner_preconditions():
    """planner.cpp:51-57: m >= c + 2 and m <= n are PlanErrors."""
    g = to_array([("h", (0,), ())])
    with pytest.raises(engine.PlanError):
        global_stages(6, 3, 4, g)
    with pytest.raises(engine.PlanError):
        global_stages(6, 2, 7, g)


def test_single_stage_when_m_equals_n(golden):
    for rec in golden["plans"]:
        if rec["m"] == rec["n"]:
            assert len(rec["stages"]) == 1
            got = global_stages(rec["n"], rec["c"], rec["m"], _circ(golden, rec["circuit"]))
            assert len(got) == 1
