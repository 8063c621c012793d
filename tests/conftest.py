"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree
libbitlamb_b200.so; everything else runs on the CPU."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def _make_oracle():
    """Build the checkers if missing (the reference-library build needs
    /root/reference, present only in the development container)."""
    odir = os.path.join(ROOT, "oracle")
    want = ["liboracle_f32.so", "liboracle_f64.so"]
    if not all(os.path.exists(os.path.join(odir, w)) for w in want):
        subprocess.run(["make", "-s", "-C", odir, "oracle"], check=True)
    ref = os.path.join(odir, "_ref", "libbitlamb_ref.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", odir, "ref"], check=True)


_make_oracle()


def have_ref() -> bool:
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbitlamb_ref.so"))


@pytest.fixture(scope="session")
def bl():
    """The product module; fails loudly (no fallback) if the library or GPU is missing."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_2104_06069_b200 import bitlamb

    return bitlamb
