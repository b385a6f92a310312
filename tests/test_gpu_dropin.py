"""Drop-in check: the REFERENCE's own C++ unit tests and acceptance gate,
compiled unmodified against include/qzsim + libqzsim_b200.so
(tests/cpp/build_reference_tests.sh, run where /root/reference exists; the
binaries travel with the repo snapshot).  Skipped where they were not built."""
import os
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "build" / "reftests"

UNIT = ["test_codec", "test_store", "test_planner", "test_device", "test_pipeline", "test_gates",
        "test_oracle"]


def _run(name, args=(), timeout=900):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (tests/cpp/build_reference_tests.sh)")
    env = dict(os.environ, LD_LIBRARY_PATH=str(ROOT / "paper_2309_16979_b200" / "lib"))
    p = subprocess.run([str(exe), *args], capture_output=True, text=True, timeout=timeout,
                       cwd="/tmp", env=env)
    return p


@pytest.mark.parametrize("name", UNIT)
def test_reference_unit_suite(name):
    p = _run(name)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("criterion", ["1", "2", "3", "4", "5", "6", "7", "8"])
def test_reference_acceptance(criterion):
    p = _run("acceptance", [criterion], timeout=1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
