"""Parity at the benchmarked scale.

bench.py times BERT-Large (d = 336,226,108, 302 tensors) through
``Optimizer.step_resident``: gradients written straight into the library's
device gradient buffers (``bl_optimizer_grad_buffer``), the dynamic tile
counter and the boundary-first tile order.  These tests run exactly that path
and compare it BIT-EXACTLY with the f32 oracle (oracle/liboracle_f32.so, the
restatement pinned to the reference) on the same inputs:

* BERT-Large, n = 1: two warmup LAMB steps, the freeze, three compression
  steps (the bench's warm start);
* BERT-Base with 4 simulated ranks (config 2): warmup, freeze, compression;
* BERT-Large with 8 simulated ranks: one warmup step (freeze) and one
  compression step -- every worker packet, server packet and residual.

Compared every step: the per-layer trace (c, r, ||v||, pre-clip ratio) and
the compressed flag; at the end: x, m, v, v_frozen, per-layer scalars, every
worker/server packet (serialize() bytes), every worker/server residual.
Reference: comm_sim.cpp:120-203, optimizers.cpp:140-177,202-224,231-332.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2104_06069_b200 import layouts

pytestmark = pytest.mark.gpu


def _grad_sigma(sizes, seed=1):
    """bench.py's per-tensor gradient scale 10^(-4+2u)."""
    u = np.random.default_rng(seed).random(len(sizes))
    return 10.0 ** (-4 + 2 * u)


def _same(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if not np.array_equal(a, b):
        bad = np.flatnonzero(a != b)
        raise AssertionError(f"{what}: {bad.size} of {a.size} differ, first at {bad[:5]}: "
                             f"{a.ravel()[bad[:5]]} vs {b.ravel()[bad[:5]]}")


def run_scale(bl, layout, n, warmup, compressed, seed=1):
    import torch

    sizes = layouts.sizes(layout)
    d = sum(sizes)
    steps = warmup + compressed
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    cl = bl.SimCluster(n, d, device=0, stream=stream.cuda_stream)
    opt = bl.Optimizer("onebit_lamb", layout, bl.HyperParams(total_steps=steps + 1, warmup_steps=warmup),
                       cl)
    ocl = O.Cluster("f32", n, d)
    oopt = O.Optimizer("f32", "onebit_lamb", sizes, O.HyperParams(total_steps=steps + 1, warmup_steps=warmup))

    gen = torch.Generator(device=dev).manual_seed(1000 + seed)
    x0 = torch.randn(d, generator=gen, device=dev) * 0.02
    opt.set("x", x0.cpu().numpy())
    oopt.set("x", x0.cpu().numpy())
    del x0
    sig = torch.from_numpy(np.repeat(_grad_sigma(sizes, seed), sizes).astype(np.float32)).to(dev)
    views = [opt.grad_tensor(i) for i in range(n)]
    host = np.empty((n, d), dtype=np.float32)
    for t in range(steps):
        for i in range(n):  # gradients written into the library's device buffers (bench.py path)
            g = torch.randn(d, generator=gen, device=dev) * sig
            views[i].copy_(g)
            host[i] = g.cpu().numpy()
            del g
        tr = opt.step_resident(t, 1e-3, trace=True)
        otr = oopt.step(host, t, 1e-3, ocl)
        assert tr.compressed == otr["compressed"] == (t >= warmup), t
        for k in ("c", "r", "v_norm", "v_ratio_preclip"):
            _same(getattr(tr, k), otr[k], f"trace {k} t={t}")
    del host
    assert opt.frozen() and oopt.frozen
    for k in ("x", "m", "v", "v_frozen"):
        _same(opt.get(k), oopt.get(k), k)
    sc, osc = opt.scalars(), oopt.scalars()
    for k in ("c_avg", "r_prev", "scale_coeff"):
        _same(sc[k], osc[k], k)
    for j in range(n):
        assert cl.server_packet(j) == ocl.server_packet(j), f"server packet {j}"
        _same(cl.server_error(j), ocl.server_error(j), f"serr {j}")
    for i in range(n):
        for j in range(n):
            assert cl.packet(i, j) == ocl.packet(i, j), f"worker packet {i}->{j}"
        _same(cl.worker_error(i), ocl.worker_error(i), f"werr {i}")
    assert cl.ledger().__dict__ == ocl.ledger()
    return opt, cl


def test_bert_large_n1_bench_path_bitexact(bl):
    """BENCH's configuration itself: BERT-Large, one rank, 2 warmup steps,
    the freeze, 3 compression steps through step_resident."""
    run_scale(bl, layouts.bert_large(), 1, warmup=2, compressed=3)


def test_bert_base_sim4_bitexact(bl):
    """Config 2: BERT-Base with 4 simulated ranks in one GPU's HBM."""
    run_scale(bl, layouts.bert_base(), 4, warmup=2, compressed=2, seed=2)


def test_bert_large_sim8_one_step_bitexact(bl):
    """BERT-Large with 8 simulated ranks (c = 42,028,264, live padding of 4):
    one warmup step that freezes, then one compression step; all 64 worker
    packets, 8 server packets and all residuals."""
    run_scale(bl, layouts.bert_large(), 8, warmup=1, compressed=1, seed=3)
