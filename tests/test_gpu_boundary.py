"""The drop-in boundary's remaining contracts, on the GPU through the C-ABI.

* Strict mode = Optimizer::check_gradients before any mutation
  (optimizers.cpp:99-117, called first at :337): a non-finite gradient raises
  the reference's exact message (layer NAMES included, LayerSpec) and leaves
  x, m, v, v_frozen, every residual, every packet, the scalars and the ledger
  bit-unchanged; the run then continues bit-exactly with the f32 oracle, which
  rejected the same step the same way.
* The free functions compress_with_feedback (compression.hpp:106-118) and
  compute_scales / apply_scaling / remove_scaling (fusion.hpp:92-102), with the
  reference's known-answer tests re-hosted (test_compression.cpp:47-205,
  test_fusion.cpp:90-153) and bit-exact against the f32 oracle.
* SimCluster::config() / step_count() (comm_sim.hpp:105,108).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

SIZES = [3000, 2, 1024, 1023, 5000, 3, 4096 * 3 + 17]
NAMES = ["emb.word", "emb.ln.b", "l0.qkv.b", "l0.out.b", "l0.inter.w", "cls.bias", "pool.w"]


def _same(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape and np.array_equal(a, b), what


def _snapshot(opt, cl):
    st = {k: opt.get(k) for k in ("x", "m", "v", "v_frozen", "m_prev")}
    st.update({f"werr{i}": cl.worker_error(i) for i in range(cl.n_workers())})
    st.update({f"serr{j}": cl.server_error(j) for j in range(cl.n_workers())})
    if cl.ledger().compressed_collectives:
        st.update({f"spk{j}": np.frombuffer(cl.server_packet(j), np.uint8) for j in range(cl.n_workers())})
    for k, v in opt.scalars().items():
        st[k] = v
    st["ledger"] = np.array(list(cl.ledger().__dict__.values()))
    return st


@pytest.mark.parametrize("n", [1, 4])
def test_strict_mode_rejects_before_any_mutation(bl, n):
    d = sum(SIZES)
    steps, warm = 12, 4
    hp = bl.HyperParams(total_steps=steps + 4, warmup_steps=warm)
    cl = bl.SimCluster(n, d)
    opt = bl.Optimizer("onebit_lamb", list(zip(NAMES, SIZES)), hp, cl, strict=True)
    ocl = O.Cluster("f32", n, d)
    oopt = O.Optimizer("f32", "onebit_lamb", SIZES, O.HyperParams(total_steps=steps + 4, warmup_steps=warm))
    rng = np.random.default_rng(100 + n)
    x0 = (rng.standard_normal(d) * 0.02).astype(np.float32)
    opt.set("x", x0)
    oopt.set("x", x0)
    sig = np.repeat(10.0 ** (-4 + 2 * rng.random(len(SIZES))), SIZES).astype(np.float32)
    for t in range(steps):
        g = (rng.standard_normal((n, d)) * sig).astype(np.float32)
        if t in (2, warm - 1, 7):  # warmup, the freezing step, compression stage
            bad = g.copy()
            w = n - 1
            bad[w, 3000 + 2 + 1024 + 5] = np.nan if t != 7 else -np.inf  # layer l0.out.b
            before = _snapshot(opt, cl)
            with pytest.raises(bl.NumericalError) as ei:
                opt.step(bad, t, 1e-3)
            assert str(ei.value) == f"non-finite gradient at step {t}, worker {w}, layer 'l0.out.b'"
            after = _snapshot(opt, cl)
            for k in before:
                _same(after[k], before[k], f"{k} changed by the rejected step t={t}")
            assert opt.frozen() == (t >= warm)
            with pytest.raises(O.OracleError, match="non-finite gradient"):
                oopt.step(bad, t, 1e-3, ocl)
        tr = opt.step(g, t, 1e-3)
        otr = oopt.step(g, t, 1e-3, ocl)
        for k in ("c", "r", "v_norm", "v_ratio_preclip"):
            _same(getattr(tr, k), otr[k], f"trace {k} t={t}")
    for k in ("x", "m", "v", "v_frozen"):
        _same(opt.get(k), oopt.get(k), k)
    for i in range(n):
        _same(cl.worker_error(i), ocl.worker_error(i), f"werr {i}")
        assert cl.server_packet(i) == ocl.server_packet(i)
    assert cl.ledger().__dict__ == ocl.ledger()


def test_strict_mode_asynchronous_steps_roll_back(bl):
    """Steps enqueued without a trace after a rejected one are skipped on the
    device; the next synchronizing call raises the FIRST failure and the state
    is the state before it."""
    import torch

    d = sum(SIZES)
    hp = bl.HyperParams(total_steps=20, warmup_steps=2)
    cl = bl.SimCluster(1, d)
    opt = bl.Optimizer("onebit_lamb", list(zip(NAMES, SIZES)), hp, cl, strict=True)
    ocl = O.Cluster("f32", 1, d)
    oopt = O.Optimizer("f32", "onebit_lamb", SIZES, O.HyperParams(total_steps=20, warmup_steps=2))
    rng = np.random.default_rng(5)
    gs = [(rng.standard_normal((1, d)) * 1e-3).astype(np.float32) for _ in range(8)]
    for t in range(4):
        opt.step(gs[t], t, 1e-3)
        oopt.step(gs[t], t, 1e-3, ocl)
    before = _snapshot(opt, cl)
    bad = gs[4].copy()
    bad[0, 0] = np.nan
    opt.step(bad, 4, 1e-3, trace=False)           # rejected on the device
    opt.step(gs[5], 5, 1e-3, trace=False)         # skipped (gate closed)
    opt.step(torch.from_numpy(gs[6]).cuda(), 6, 1e-3, trace=False)
    with pytest.raises(bl.NumericalError, match=r"at step 4, worker 0, layer 'emb.word'"):
        cl.synchronize()
    after = _snapshot(opt, cl)
    for k in before:
        _same(after[k], before[k], k)
    for t in (4, 5, 6, 7):  # the run resumes from the state before step 4
        tr = opt.step(gs[t], t, 1e-3)
        otr = oopt.step(gs[t], t, 1e-3, ocl)
        _same(tr.c, otr["c"], f"c t={t}")
    _same(opt.get("x"), oopt.get("x"), "x")


def test_fused_mode_reports_layer_name_after_the_step(bl):
    """Default (fused) mode: the check rides in the first kernel that reads the
    gradient and is reported by the synchronizing call, with the layer name."""
    d = sum(SIZES)
    cl = bl.SimCluster(2, d)
    opt = bl.Optimizer("onebit_lamb", list(zip(NAMES, SIZES)), bl.HyperParams(total_steps=8, warmup_steps=2), cl)
    g = np.zeros((2, d), np.float32)
    for t in range(3):
        opt.step(g, t, 1e-3)
    g[1, d - 1] = np.inf
    with pytest.raises(bl.NumericalError, match=r"non-finite gradient at step 3, worker 1, layer 'pool.w'"):
        opt.step(g, 3, 1e-3)


def test_layer_names_and_cluster_accessors(bl):
    d = sum(SIZES)
    cl = bl.SimCluster(3, d, compressor="onebit", baseline_bits_per_element=32, verify_compensation=True,
                       compensation_tolerance=2.0 ** -20)
    opt = bl.Optimizer("onebit_lamb", list(zip(NAMES, SIZES)), bl.HyperParams(total_steps=8, warmup_steps=2), cl)
    assert [opt.layer_name(i) for i in range(len(NAMES))] == NAMES
    cfg = cl.config()
    assert cfg["n_workers"] == 3 and cfg["dim"] == d and cfg["baseline_bits_per_element"] == 32
    assert cfg["verify_compensation"] and cfg["compensation_tolerance"] == 2.0 ** -20
    assert cl.step_count() == 0
    g = (np.random.default_rng(0).standard_normal((3, d)) * 1e-3).astype(np.float32)
    for t in range(4):  # comm_sim.cpp:197,230: one per collective, lossless or compressed
        opt.step(g, t, 1e-3)
        assert cl.step_count() == t + 1
    cl.compressed_allreduce(g)
    assert cl.step_count() == 5


# ---------------------------------------------------------------------------
# compress_with_feedback (compression.hpp:106-118)
# ---------------------------------------------------------------------------
def test_compress_with_feedback_known_answers(bl):
    # test_compression.cpp:47-57: [2,-1,0.5,-0.5] -> S = 1, signs + - + -
    v = np.array([2.0, -1.0, 0.5, -0.5], np.float32)
    dl = np.zeros(4, np.float32)
    wire, dec = bl.compress_with_feedback(v, dl)
    assert wire[0] & 0xF == 0b0101 and np.frombuffer(wire[1:], np.float32)[0] == 1.0
    _same(dec, [1, -1, 1, -1], "dec")
    _same(dl, v - dec, "delta")
    # :59-63 zero input -> S = 0 and exact zeros
    wire, dec = bl.compress_with_feedback(np.zeros(5, np.float32), np.zeros(5, np.float32))
    assert np.frombuffer(wire[1:], np.float32)[0] == 0.0 and not dec.any()
    # :65-68 constant magnitude is lossless
    v = np.array([3.0, -3.0, 3.0], np.float32)
    dl = np.zeros(3, np.float32)
    _, dec = bl.compress_with_feedback(v, dl)
    _same(dec, v, "lossless")
    assert not dl.any()
    # :84-100 single element exact; [1, 0] -> dec [0.5, 0.5], delta [0.5, -0.5]
    dl = np.zeros(1, np.float32)
    _, dec = bl.compress_with_feedback(np.array([0.3], np.float32), dl)
    _same(dec, np.array([0.3], np.float32), "single")
    _same(dl, [0.0], "single delta")
    dl = np.zeros(2, np.float32)
    _, dec = bl.compress_with_feedback(np.array([1.0, 0.0], np.float32), dl)
    _same(dec, [0.5, 0.5], "dec")
    _same(dl, [0.5, -0.5], "delta")
    # :102-112 identity keeps delta at zero; the message is v + es*delta
    dl = np.array([0.25, -1.0], np.float32)
    wire, dec = bl.compress_with_feedback(np.array([1.0, 2.0], np.float32), dl, kind="identity", error_scale=0.5)
    assert wire is None
    _same(dec, [1.125, 1.5], "identity message")
    _same(dl, [0.0, 0.0], "identity delta")
    # :169-191 golden wire bytes
    v = np.array([1, -1, -1, 1, 1, 1, -1, 1, -1, 1], np.float32)
    wire, _ = bl.compress_with_feedback(v, np.zeros(10, np.float32))
    assert wire == bytes([0b10111001, 0b00000010, 0x00, 0x00, 0x80, 0x3F])


@pytest.mark.parametrize("d", [1, 7, 4096, 4097, 100003])
@pytest.mark.parametrize("es", [1.0, 0.75])
def test_compress_with_feedback_bitexact_vs_oracle(bl, d, es):
    rng = np.random.default_rng(d)
    v = rng.standard_normal(d).astype(np.float32)
    dl = (rng.standard_normal(d) * 0.3).astype(np.float32)
    odl = dl.copy()
    for _ in range(3):  # carried residual over several calls
        wire, dec = bl.compress_with_feedback(v, dl, error_scale=es)
        owire, oscale, odec, odl = O.compress_with_feedback("f32", v, odl, error_scale=es)
        assert wire == owire
        _same(dec, odec, "decompressed")
        _same(dl, odl, "delta")
        v = rng.standard_normal(d).astype(np.float32)


def test_compress_with_feedback_nonfinite_leaves_delta(bl):
    """compression.cpp:56-58 throws before the residual update."""
    v = np.array([1.0, np.nan, 2.0], np.float32)
    dl = np.array([0.1, 0.2, 0.3], np.float32)
    with pytest.raises(bl.InvalidArgument, match="not finite"):
        bl.compress_with_feedback(v, dl)
    _same(dl, np.array([0.1, 0.2, 0.3], np.float32), "delta after the throw")
    with pytest.raises(bl.DimensionError):
        bl.compress_with_feedback(np.zeros(3, np.float32), np.zeros(2, np.float32))


# ---------------------------------------------------------------------------
# compute_scales / apply_scaling / remove_scaling (fusion.hpp:92-102)
# ---------------------------------------------------------------------------
def test_compute_scales_known_answer(bl):
    """test_fusion.cpp:90-100: magnitudes 0.1 and 0.4 -> reference 0.25,
    coeff 2.5 and 0.625."""
    m = np.concatenate([np.full(3, -0.1), np.full(5, 0.4)]).astype(np.float32)
    coeff, ref = bl.compute_scales(m, [3, 5])
    s = [O.canonical_sum("f32", m[:3], 0) / 3, O.canonical_sum("f32", m[3:], 0) / 5]
    want_ref = (s[0] + s[1]) / 2
    assert ref == want_ref
    _same(coeff, [want_ref / s[0], want_ref / s[1]], "coeff")
    assert abs(coeff[0] - 2.5) < 1e-6 and abs(coeff[1] - 0.625) < 1e-6
    # floored magnitude: an all-zero layer gets s = floor
    coeff, ref = bl.compute_scales(np.zeros(4, np.float32), [2, 2], floor=1e-3)
    assert ref == 1e-3 and np.array_equal(coeff, [1.0, 1.0])
    with pytest.raises(bl.InvalidArgument, match="floor must be positive"):
        bl.compute_scales(np.zeros(4, np.float32), [4], floor=0.0)


def test_compute_scales_bitexact_canonical_order(bl):
    rng = np.random.default_rng(9)
    sizes = [1, 4096, 4097, 70001, 3]
    m = (rng.standard_normal(sum(sizes)) * 10.0 ** rng.uniform(-5, 0, sum(sizes))).astype(np.float32)
    coeff, ref = bl.compute_scales(m, sizes)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    mag = []
    for l in range(len(sizes)):  # vector_ops.cpp:41-44 over the canonical tile-tree sum
        seg = m[offs[l]:offs[l + 1]]
        mean = O.canonical_sum("f32", seg, 0) / len(seg)
        mag.append(max(mean, 1e-12))
    want_ref = 0.0
    for s in mag:
        want_ref += s
    want_ref /= len(mag)
    assert ref == want_ref
    _same(coeff, [want_ref / s for s in mag], "coeff")


def test_apply_remove_scaling(bl):
    rng = np.random.default_rng(4)
    sizes = [5, 4099, 1, 300]
    x = rng.standard_normal(sum(sizes)).astype(np.float32)
    coeff = np.array([2.5, 0.625, 3.0, 1.0 / 3.0])
    up = bl.apply_scaling(x, sizes, coeff)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    for l in range(len(sizes)):  # kernels::scale: x *= c (fp32: the factor rounded once)
        seg = slice(offs[l], offs[l + 1])
        _same(up[seg], x[seg] * np.float32(coeff[l]), f"apply layer {l}")
    down = bl.remove_scaling(up, sizes, coeff)
    for l in range(len(sizes)):
        seg = slice(offs[l], offs[l + 1])
        _same(down[seg], up[seg] * np.float32(1.0 / coeff[l]), f"remove layer {l}")
    # power-of-two scales round-trip exactly (test_fusion.cpp:124-153)
    c2 = np.array([2.0, 0.5, 4.0, 0.25])
    _same(bl.remove_scaling(bl.apply_scaling(x, sizes, c2), sizes, c2), x, "round trip")
    with pytest.raises(bl.DimensionError):
        bl.apply_scaling(x, sizes, coeff[:2])


def test_graph_replay_follows_the_lr_schedule(bl):
    """The steady-state compression step is replayed from a captured CUDA
    graph; its lr is staged into device memory before each replay.  A
    per-step lr (schedule.cpp-style decay) must still give the oracle's
    trajectory bit for bit, at n = 1 and with 4 simulated ranks."""
    for n in (1, 4):
        d = sum(SIZES)
        steps, warm = 12, 3
        cl = bl.SimCluster(n, d)
        opt = bl.Optimizer("onebit_lamb", SIZES, bl.HyperParams(total_steps=steps, warmup_steps=warm), cl)
        ocl = O.Cluster("f32", n, d)
        oopt = O.Optimizer("f32", "onebit_lamb", SIZES, O.HyperParams(total_steps=steps, warmup_steps=warm))
        rng = np.random.default_rng(77 + n)
        x0 = (rng.standard_normal(d) * 0.02).astype(np.float32)
        opt.set("x", x0)
        oopt.set("x", x0)
        for t in range(steps):
            lr = 1e-3 * (0.7 ** t)
            g = (rng.standard_normal((n, d)) * 1e-3).astype(np.float32)
            tr = opt.step(g, t, lr)
            otr = oopt.step(g, t, lr, ocl)
            _same(tr.c, otr["c"], f"c t={t} n={n}")
        _same(opt.get("x"), oopt.get("x"), f"x n={n}")
