"""The C++ drop-in path on the GPU: tests/cpp/facade_demo.cpp, built against
include/bitlamb_b200.hpp and libbitlamb_b200.so, drives SimCluster and the
1-bit LAMB Optimizer like the reference's callers do.  Its outputs are
replayed on the f32 oracle and must match bit for bit."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def f32(path):
    return np.fromfile(path, dtype=np.float32)


def test_cpp_facade_on_gpu_matches_oracle(tmp_path):
    from paper_2104_06069_b200 import build

    lib = build.build()
    exe = tmp_path / "facade_demo"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "facade_demo.cpp"),
                    f"-L{os.path.dirname(lib)}", "-lbitlamb_b200",
                    f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "facade ok" in r.stdout, r.stdout + r.stderr
    assert "DimensionError ok" in r.stdout and "frozen=1" in r.stdout

    n, d = 4, 10007
    oc = O.Cluster("f32", n, d)
    for call in range(3):
        x = f32(tmp_path / f"ar_in{call}.bin").reshape(n, d)
        np.testing.assert_array_equal(f32(tmp_path / f"ar_out{call}.bin"), oc.compressed_allreduce(x))

    sizes = [3000, 2, 1023, 4099]
    dd = sum(sizes)
    opt = O.Optimizer("f32", "onebit_lamb", sizes, O.HyperParams(total_steps=12, warmup_steps=4))
    ocl = O.Cluster("f32", 2, dd)
    opt.set("x", f32(tmp_path / "opt_x0.bin"))
    for t in range(12):
        tr = opt.step(f32(tmp_path / f"opt_g{t}.bin").reshape(2, dd), t, 1e-3, ocl)
        np.testing.assert_array_equal(f32(tmp_path / f"opt_c{t}.bin"), tr["c"].astype(np.float32))
    np.testing.assert_array_equal(f32(tmp_path / "opt_x.bin"), opt.get("x"))
    np.testing.assert_array_equal(f32(tmp_path / "opt_v.bin"), opt.get("v"))
