"""CPU suite: the drop-in boundary without a GPU.

* libbitlamb_b200.so loads and exports every entry point include/bitlamb_b200.h
  declares (the symbols a cgo/ctypes/JNI binding would bind).
* Host-only entry points work (volume_reduction, hparams defaults) and agree
  with the reference; device entry points fail loudly (no CPU fallback).
* The C++ facade (include/bitlamb_b200.hpp) compiles, links and maps status
  codes to the reference's exception classes.
* The BERT layer tables match SURVEY.md Appendix B.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bitlamb_b200.h")
LIB = os.path.join(ROOT, "paper_2104_06069_b200", "libbitlamb_b200.so")


@pytest.fixture(scope="module")
def built():
    sys.path.insert(0, ROOT)
    from paper_2104_06069_b200 import build

    build.build()
    return LIB


def declared_functions() -> list[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bl_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("bl_cluster_create", "bl_cluster_compressed_allreduce", "bl_cluster_lossless_allreduce",
                 "bl_optimizer_create", "bl_optimizer_step", "bl_volume_reduction", "bl_last_error"):
        assert must in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol(built):
    so = C.CDLL(built)
    missing = [n for n in declared_functions() if not hasattr(so, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bl_[a-z0-9_]+)", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_entry_points_match_reference(built):
    from oracle import oracle as O
    from paper_2104_06069_b200 import bitlamb as bl

    for w in (0.0, 0.167, 0.193, 0.5, 1.0):
        assert bl.volume_reduction(w, 16, 1.0) == O.volume_reduction("f64", w, 16, 1.0)
    with pytest.raises(bl.InvalidArgument):
        bl.volume_reduction(1.5, 16, 1.0)
    hp = bl._HParams()
    bl.lib.bl_hparams_default(C.byref(hp))
    ref = bl.HyperParams()
    for k in ("beta1", "beta2", "beta3", "eta", "c_min", "c_max", "r_min", "r_max", "r_threshold",
              "weight_decay", "division_floor"):
        assert getattr(hp, k) == getattr(ref, k) == getattr(O.HyperParams(), k)


def test_device_paths_fail_loudly_without_gpu(built):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2104_06069_b200 import bitlamb as bl

    with pytest.raises(bl.CudaError):
        bl.SimCluster(2, 10)


def test_cpp_facade_compiles_and_maps_errors(built, tmp_path):
    src = tmp_path / "facade.cpp"
    src.write_text(r'''
#include <cstdio>
#include <vector>
#include "bitlamb_b200.hpp"
int main() {
  using namespace bitlamb_b200;
  std::printf("vr=%.6f\n", volume_reduction(0.167, 16, 1.0));
  try { volume_reduction(2.0, 16, 1.0); } catch (const std::invalid_argument& e) { std::printf("invalid_argument\n"); }
  try {
    SimCluster::Config cfg; cfg.n_workers = 2; cfg.dim = 10;
    SimCluster c(cfg);
    std::vector<std::vector<float>> in(2, std::vector<float>(10, 1.0f));
    auto out = c.compressed_allreduce(in);
    std::printf("ran %zu\n", out.size());
  } catch (const CudaError& e) { std::printf("CudaError\n"); }
  return 0;
}
''')
    exe = tmp_path / "facade"
    lib_dir = os.path.dirname(built)
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include",
                    str(src), f"-L{lib_dir}", "-lbitlamb_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60).stdout
    assert "vr=4.564907" in out and "invalid_argument" in out
    assert "CudaError" in out or "ran 10" in out


def test_bert_layouts_match_survey():
    from paper_2104_06069_b200 import layouts

    base, large = layouts.bert_base(), layouts.bert_large()
    assert len(base) == 158 and sum(layouts.sizes(base)) == 110_106_428
    assert len(large) == 302 and sum(layouts.sizes(large)) == 336_226_108
    assert min(layouts.sizes(large)) == 2 and max(layouts.sizes(large)) == 31_254_528
    assert sum(layouts.CONFIG1) == 8_000_003 and len(layouts.CONFIG1) == 16
    d = 336_226_108
    for n, c, mod in ((1, 336_226_108, 28), (2, 168_113_054, 30), (4, 84_056_527, 15), (8, 42_028_264, 8)):
        P = -(-d // n) * n
        assert P // n == c and c % 32 == mod


def test_bench_byte_model():
    sys.path.insert(0, ROOT)
    import bench

    ab = bench.algorithmic_bytes(336_226_108, 1, 1)
    total = sum(v for k, v in ab.items() if not k.startswith("w"))
    assert 44.5 < total / 336_226_108 < 45.5  # ~44.9 B/param at n=1
    ab8 = bench.algorithmic_bytes(336_226_108, 8, 1)
    assert ab8["k3_server_reduce"] < ab["k3_server_reduce"] / 7
    # owner-sharded warmup: a rank updates 1/n of the tiles
    ab4 = bench.algorithmic_bytes(336_226_108, 4, 1, share=0.25)
    assert ab4["w1_warmup_a"] == ab["w1_warmup_a"] / 4 and ab4["w2_warmup_b"] == ab["w2_warmup_b"] / 4
    assert ab4["k5_update_a"] == ab["k5_update_a"]  # the compression stage stays replicated


def test_bench_reference_arm_prints_contract_line():
    from conftest import have_ref

    if not have_ref():
        pytest.skip("oracle/_ref not built")
    env = dict(os.environ, BL_REF_THREADS="4")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--workload", "config1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "ms" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] == 4
    assert line["e2e"]["h2d_bytes_per_step"] == 0
