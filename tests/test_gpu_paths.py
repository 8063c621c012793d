"""The alternate kernel paths that the size heuristics route around, forced on
small inputs and checked bit-exact against the f32 oracle by rerunning the
optimizer parity tests of test_gpu_parity.py in a subprocess:

- "bulk": K1 through the bulk-copy pipeline for every misaligned chunk
  length (by default problems of at most 16384 K1 tiles take the register
  path, bl_kernels.cu k1_uses_bulk);
- "inline": K5/K6 general-path tiles inside the streaming kernels instead
  of k5_general / k6_general on the side stream (BL_GENERAL_SPLIT_MAX_TILES=0);
- "static": grid-stride tiles instead of the atomic tile counter.
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ENV = {
    "bulk": {"BL_K1_BULK": "all"},
    "inline": {"BL_GENERAL_SPLIT_MAX_TILES": "0"},
    "static": {"BL_STATIC_TILES": "1"},
}


@pytest.mark.parametrize("path", sorted(ENV))
def test_optimizer_parity_on_alternate_path(path):
    env = dict(os.environ, **ENV[path])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"),
           "-k", "optimizer_onebit_lamb_bitexact or misaligned_layer_full_tiles or other_variants"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert r.returncode == 0 and " passed" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
