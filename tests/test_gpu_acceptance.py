"""the reference's acceptance criteria on the B200 backend.

oracle/_ref/acceptance_b200 (tests/cpp/acceptance_b200.cpp, built by
`make -C oracle accept` where /root/reference exists) runs the reference's
toy-task training protocol — its tasks, sharding, schedule and metrics CSV —
with bitlamb_b200::SimCluster / Optimizer as the optimizer and communicator,
and checks acceptance.cpp's criteria 1-10 plus agreement with the
reference's own fp64 trainer (criterion 11)."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def test_reference_acceptance_criteria_on_b200(bl):
    if not os.path.exists(EXE):
        if os.path.isdir("/root/reference/proj/src"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref", "accept"], check=True)
        else:
            pytest.fail("oracle/_ref/acceptance_b200 was not built (run __graft_entry__.build() "
                        "where /root/reference exists)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(EXE))
    out = r.stdout + r.stderr
    verdicts = re.findall(r"^\[(PASS|FAIL)\] criterion (\d+): ", r.stdout, re.M)
    assert [int(k) for _, k in verdicts] == list(range(1, 12)), out
    assert all(v == "PASS" for v, _ in verdicts), out
    assert r.returncode == 0 and "all criteria passed" in r.stdout, out
