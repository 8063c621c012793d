"""GPU parity suite: the sm_100a path through the C-ABI against the checkers.

* vs oracle f32 (liboracle_f32.so): BIT-EXACT — packets, scales, results,
  worker/server residuals, optimizer state and traces, every step.
* vs the reference library (oracle/_ref, fp64) on identical fp32-representable
  inputs: sign packets bit-exact on a single collective, scales within 1 fp32
  ulp, multi-step trajectories within the fp32 tolerances stated below.
* the reference's own known-answer tests re-hosted on the GPU path
  (test_compression.cpp, test_comm_sim.cpp, test_optimizers.cpp).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2104_06069_b200 import layouts

from conftest import have_ref

pytestmark = pytest.mark.gpu


def rnd(shape, seed, sigma=1.0):
    return (np.random.default_rng(seed).standard_normal(shape) * sigma).astype(np.float32)


def assert_same(a, b, what=""):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if not np.array_equal(a, b):
        bad = np.nonzero(a != b)[0]
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[:5]}: "
                             f"{a[bad[:5]]} vs {b[bad[:5]]}")


# ---------------------------------------------------------------------------
# Compressed allreduce (comm_sim.cpp:120-203)
# ---------------------------------------------------------------------------
CASES = [(1, 1), (1, 6), (2, 4), (2, 5), (3, 10), (4, 23), (8, 37), (5, 16), (4, 4096),
         (4, 10000), (2, 8193), (3, 100003), (8, 65536 * 3 + 5), (4, layouts.CONFIG1[0] + 3)]


@pytest.mark.parametrize("n,d", CASES)
def test_compressed_allreduce_bitexact_vs_oracle_f32(bl, n, d):
    g = bl.SimCluster(n, d)
    o = O.Cluster("f32", n, d)
    for step in range(4):
        x = rnd((n, d), 1000 * n + d + step)
        if step == 2:
            x[:, : min(d, 7)] = 0.0  # exact zeros: sign of 0 is +1 (compression.cpp:50)
        es = 1.0 if step < 3 else 0.75  # experimental scaled carry (:181)
        a = g.compressed_allreduce(x, error_scale=es)
        b = o.compressed_allreduce(x, error_scale=es)
        assert_same(a, b, f"result step {step}")
        for i in range(n):
            assert_same(g.worker_error(i), o.worker_error(i), f"werr {i} step {step}")
            assert_same(g.server_error(i), o.server_error(i), f"serr {i} step {step}")
            assert g.server_packet(i) == o.server_packet(i)
            for j in range(n):
                assert g.packet(i, j) == o.packet(i, j), (step, i, j)
    led = g.ledger()
    assert led.__dict__ == o.ledger()


@pytest.mark.skipif(not have_ref(), reason="reference library not built")
@pytest.mark.parametrize("n,d", [(1, 6), (2, 5), (4, 23), (8, 37), (4, 10000), (3, 100003)])
def test_single_collective_packets_vs_reference(bl, n, d):
    """Identical fp32 inputs: sign bytes bit-exact against the fp64 reference's
    serialize(); scales equal static_cast<float>(S_ref) within 1 ulp."""
    x = rnd((n, d), 77 + d)
    g = bl.SimCluster(n, d)
    r = O.Cluster("ref", n, d)
    a = g.compressed_allreduce(x)
    b = r.compressed_allreduce(x.astype(np.float64))
    nb = (g.chunk_len + 7) // 8
    for i in range(n):
        for j in range(n):
            pg, pr = g.packet(i, j), r.packet(i, j)
            assert pg[:nb] == pr[:nb], (i, j)
            sg = np.frombuffer(pg[nb:], np.float32)[0]
            sr = np.frombuffer(pr[nb:], np.float32)[0]
            assert abs(int(sg.view(np.int32)) - int(sr.view(np.int32))) <= 1
    # second phase sees identical packets, so the results agree to fp32 rounding
    np.testing.assert_allclose(a, b, rtol=2e-7, atol=0)


def test_identity_compressor_collapses_to_average(bl):
    """test_comm_sim.cpp:106-134 (identity == lossless, residuals stay 0)."""
    for n in (1, 2, 3, 4, 8):
        for d in (1, 5, 16, 37):
            x = rnd((n, d), 1000 + n * 100 + d)
            a = bl.SimCluster(n, d, compressor="identity").compressed_allreduce(x)
            b = bl.SimCluster(n, d, compressor="identity").lossless_allreduce(x)
            assert_same(a, b)
            assert_same(b, O.Cluster("f32", n, d).lossless_allreduce(x))


def test_lossless_allreduce_matches_reference_kat(bl):
    """test_comm_sim.cpp:53-73."""
    c = bl.SimCluster(2, 2, compressor="identity")
    assert_same(c.lossless_allreduce(np.array([[1, 2], [3, 4]], np.float32)), [2.0, 3.0])
    c = bl.SimCluster(3, 1, compressor="identity")
    assert_same(c.lossless_allreduce(np.array([[3], [6], [9]], np.float32)), [6.0])


def test_two_worker_hand_scripted(bl):
    """test_comm_sim.cpp:163-222 restated in fp32: n=2, d=4 gather/average/scatter."""
    n, d, ch = 2, 4, 2
    x = rnd((n, d), 4242)
    c = bl.SimCluster(n, d)
    out = c.compressed_allreduce(x)
    wd = np.zeros((n, d), np.float32)
    sd = np.zeros((n, ch), np.float32)
    sent = {}
    for i in range(n):
        for j in range(n):
            corr = x[i, j * ch:(j + 1) * ch] + wd[i, j * ch:(j + 1) * ch]
            s = np.float32(np.abs(corr.astype(np.float64)).sum() / ch)
            dec = np.where(corr >= 0, s, -s).astype(np.float32)
            wd[i, j * ch:(j + 1) * ch] = corr - dec
            sent[i, j] = dec
    exp = np.zeros(d, np.float32)
    for j in range(n):
        avg = np.float32((sent[0, j].astype(np.float64) + sent[1, j]) * 0.5)
        corr = avg + sd[j]
        s = np.float32(np.abs(corr.astype(np.float64)).sum() / ch)
        dec = np.where(corr >= 0, s, -s).astype(np.float32)
        sd[j] = corr - dec
        exp[j * ch:(j + 1) * ch] = dec
    assert_same(out, exp)
    for i in range(n):
        assert_same(c.worker_error(i), wd[i])
        assert_same(c.server_error(i), sd[i])


def test_wire_layout_golden_bytes(bl):
    """test_compression.cpp:169-191: + - - + + + - + | - +  -> b9 02 | 00 00 80 3f.
    A 1-worker cluster's worker packet is compress_with_feedback(v, 0)."""
    v = np.array([1, -1, -1, 1, 1, 1, -1, 1, -1, 1], np.float32)
    c = bl.SimCluster(1, 10)
    c.compressed_allreduce(v[None, :])
    assert c.packet(0, 0) == bytes([0b10111001, 0b00000010, 0x00, 0x00, 0x80, 0x3F])


def test_compress_known_answers(bl):
    """test_compression.cpp:47-100 through a 1-worker cluster."""
    c = bl.SimCluster(1, 4)
    c.compressed_allreduce(np.array([[2.0, -1.0, 0.5, -0.5]], np.float32))
    p = c.packet(0, 0)
    assert p[0] & 0xF == 0b0101 and np.frombuffer(p[1:], np.float32)[0] == 1.0
    c = bl.SimCluster(1, 3)
    out = c.compressed_allreduce(np.zeros((1, 3), np.float32))
    assert_same(out, np.zeros(3, np.float32))
    assert np.frombuffer(c.packet(0, 0)[1:], np.float32)[0] == 0.0
    c = bl.SimCluster(1, 2)
    c.compressed_allreduce(np.array([[1.0, 0.0]], np.float32))
    assert_same(c.worker_error(0), [0.5, -0.5])  # test_compression.cpp:84-91
    c = bl.SimCluster(1, 1)
    c.compressed_allreduce(np.array([[0.3]], np.float32))
    assert_same(c.worker_error(0), [0.0])


def test_compensation_identity_and_residual_bound(bl):
    """test_compression.cpp:114-147 on the device residuals: v + d_prev ==
    dec + d_new (to fp32 rounding) and max|d| <= 2 max|v + d_prev|."""
    n, d = 2, 257
    c = bl.SimCluster(n, d)
    prev = np.zeros((n, c.padded), np.float32)
    mx_d = mx_c = 0.0
    for step in range(50):
        x = rnd((n, d), 9000 + step, 0.5)
        xp = np.zeros((n, c.padded), np.float32)
        xp[:, :d] = x
        c.compressed_allreduce(x)
        for i in range(n):
            corr = (xp[i] + prev[i]).astype(np.float64)
            new = c.worker_error(i)
            nb = (c.chunk_len + 7) // 8
            dec = []
            for j in range(n):
                p = c.packet(i, j)
                s = np.frombuffer(p[nb:], np.float32)[0]
                bits = np.unpackbits(np.frombuffer(p[:nb], np.uint8), bitorder="little")[: c.chunk_len]
                dec.append(np.where(bits == 1, s, -s))
            dec = np.concatenate(dec).astype(np.float64)
            lhs, rhs = corr, dec + new
            den = np.maximum(np.maximum(np.abs(lhs), np.abs(dec)), 1e-300)
            assert np.all(np.abs(lhs - rhs) <= 2.0 ** -23 * den)
            mx_c = max(mx_c, np.abs(corr).max())
            mx_d = max(mx_d, np.abs(new).max())
            prev[i] = new
    assert mx_d <= 2 * mx_c


def test_verify_compensation_counts_and_fails_loudly(bl):
    """test_comm_sim.cpp:280-289 on the device: n^2 + n checks per call; an
    fp32 run needs an fp32 tolerance (2^-23), the fp64 default 1e-12 trips."""
    c = bl.SimCluster(2, 8, verify_compensation=True, compensation_tolerance=2.0 ** -23)
    for step in range(5):
        c.compressed_allreduce(rnd((2, 8), 600 + step))
    assert c.compensation_checks() == 5 * (2 * 2 + 2)
    tight = bl.SimCluster(1, 2, verify_compensation=True)  # tol 1e-12
    with pytest.raises(bl.LogicError, match="error-compensation identity violated"):
        tight.compressed_allreduce(np.array([[1.0, 1e-8]], np.float32))


def test_dimension_errors(bl):
    """test_comm_sim.cpp:261-268."""
    c = bl.SimCluster(2, 4)
    with pytest.raises(bl.DimensionError):
        c.compressed_allreduce([np.zeros(4, np.float32), np.zeros(3, np.float32)])
    with pytest.raises(bl.DimensionError):
        c.compressed_allreduce([np.zeros(4, np.float32)])
    with pytest.raises(bl.InvalidArgument):
        bl.SimCluster(0, 4)
    with pytest.raises(bl.InvalidArgument):
        bl.SimCluster(2, 0)


def test_nonfinite_input_raises(bl):
    c = bl.SimCluster(1, 2)
    with pytest.raises(bl.InvalidArgument):
        c.compressed_allreduce(np.array([[1.0, np.nan]], np.float32))


def test_ledger_with_padding(bl):
    """test_comm_sim.cpp:239-259: d=5, n=2 chunks of 3 and 2 real elements."""
    c = bl.SimCluster(2, 5)
    out = c.compressed_allreduce(rnd((2, 5), 333))
    assert out.shape == (5,)
    led = c.ledger()
    assert led.gather_bits == (3 + 32) + (2 + 32) and led.scatter_bits == led.gather_bits
    assert led.baseline_equivalent_bits == 2 * 1 * 5 * 16 and led.compressed_collectives == 1
    before = led.total_sent_bits()
    c.compressed_allreduce(rnd((2, 5), 333))
    assert c.ledger().total_sent_bits() == 2 * before


def test_endpoint_stats_match_oracle(bl):
    n, d = 3, 10000
    g = bl.SimCluster(n, d, endpoint_stats=True)
    o = O.Cluster("f32", n, d)
    for step in range(3):
        x = rnd((n, d), 11 + step)
        g.compressed_allreduce(x)
        o.compressed_allreduce(x)
    st = o.stats()
    got = np.array([[s.delta_l2, s.delta_linf, s.corrected_linf, s.max_delta_linf, s.max_corrected_linf]
                    for s in g.worker_stats() + g.server_stats()]).reshape(2, n, 5)
    np.testing.assert_array_equal(got, st)
    assert g.run_max_delta_linf() <= 2.0 * g.run_max_corrected_linf()


# ---------------------------------------------------------------------------
# Optimizer (optimizers.cpp:334-364): warmup LAMB, freeze, compression stage
# ---------------------------------------------------------------------------
def run_pair(bl, sizes, n, steps, warmup, seed, lr=1e-3, wd=0.0, scaled=False, check_every=1,
             grad_sigma=None, variant="onebit_lamb", kind="onebit"):
    hp = bl.HyperParams(total_steps=steps, warmup_steps=warmup, weight_decay=wd,
                        scaled_error_feedback=scaled)
    ohp = O.HyperParams(total_steps=steps, warmup_steps=warmup, weight_decay=wd,
                        scaled_error_feedback=scaled)
    d = sum(sizes)
    cl = bl.SimCluster(n, d, compressor=kind)
    opt = bl.Optimizer(variant, sizes, hp, cl)
    ocl = O.Cluster("f32", n, d, kind=kind)
    oopt = O.Optimizer("f32", variant, sizes, ohp)
    rng = np.random.default_rng(seed)
    x0 = (rng.standard_normal(d) * 0.02).astype(np.float32)
    opt.set("x", x0)
    oopt.set("x", x0)
    sig = grad_sigma if grad_sigma is not None else np.repeat(
        10.0 ** (-4 + 2 * rng.random(len(sizes))), sizes).astype(np.float32)
    for t in range(steps):
        g = (rng.standard_normal((n, d)) * sig).astype(np.float32)
        ta = opt.step(g, t, lr)
        tb = oopt.step(g, t, lr, ocl)
        for k in ("c", "r", "v_norm", "v_ratio_preclip"):
            assert_same(getattr(ta, k), tb[k], f"trace {k} t={t}")
        assert ta.compressed == tb["compressed"]
        if t % check_every == 0 or t == steps - 1:
            for k in ("x", "m", "v", "v_frozen", "m_prev"):
                assert_same(opt.get(k), oopt.get(k), f"{k} t={t}")
    return opt, oopt, cl, ocl


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_optimizer_onebit_lamb_bitexact_vs_oracle_f32(bl, n):
    sizes = [3000, 2, 1024, 1023, 5000, 3, 4096 * 3 + 17]
    opt, oopt, cl, ocl = run_pair(bl, sizes, n, steps=30, warmup=8, seed=5 + n)
    sc, osc = opt.scalars(), oopt.scalars()
    for k in ("c_avg", "r_prev", "scale_coeff"):
        assert_same(sc[k], osc[k], k)
    assert opt.frozen()
    for i in range(n):
        assert_same(cl.worker_error(i), ocl.worker_error(i))
        assert_same(cl.server_error(i), ocl.server_error(i))


@pytest.mark.parametrize("variant", ["lamb_basic_1bit", "onebit_adam", "lamb", "adam"])
def test_optimizer_other_variants_bitexact(bl, variant):
    """The reference's ablation/baseline variants (optimizers.cpp:140-200,
    301-303) through the same kernels."""
    run_pair(bl, [3000, 2, 1024, 4099], 2, steps=14, warmup=5, seed=21, variant=variant)


@pytest.mark.parametrize("variant", ["onebit_lamb", "lamb_basic_1bit"])
def test_optimizer_identity_compressor_bitexact(bl, variant):
    """Identity compressor inside the optimizer (the reference's lossless-collapse
    setup, test_optimizers.cpp:381-438)."""
    run_pair(bl, [5, 9, 4096 + 3], 4, steps=20, warmup=6, seed=91, variant=variant, kind="identity")


def test_optimizer_weight_decay_and_scaled_feedback(bl):
    run_pair(bl, [4000, 7, 2048], 2, steps=20, warmup=5, seed=3, wd=0.01, scaled=True)


def test_optimizer_config1_100_steps(bl):
    """SURVEY §8(d) config 1 layout (ragged, misaligned, live padding), n=4,
    100 steps; bit-exact with the f32 oracle at sampled steps and the end."""
    run_pair(bl, layouts.CONFIG1, 4, steps=100, warmup=10, seed=1, check_every=25)


@pytest.mark.skipif(not have_ref(), reason="reference library not built")
def test_optimizer_vs_reference_fp64_tolerance(bl):
    """The fp32 path against the fp64 reference library: 100 steps on a
    ragged 7-layer table, n=4.  Norm-wise drift of x relative to its motion
    and the fraction of flipped server-packet sign bits stay small."""
    sizes = [3000, 2, 1024, 1023, 5000, 3, 4096 * 3 + 17]
    n, steps, warm, d = 4, 100, 10, sum(sizes)
    hp = bl.HyperParams(total_steps=steps, warmup_steps=warm)
    rhp = O.HyperParams(total_steps=steps, warmup_steps=warm)
    cl = bl.SimCluster(n, d)
    opt = bl.Optimizer("onebit_lamb", sizes, hp, cl)
    rcl = O.Cluster("ref", n, d)
    ropt = O.Optimizer("ref", "onebit_lamb", sizes, rhp)
    rng = np.random.default_rng(0)
    x0 = (rng.standard_normal(d) * 0.02).astype(np.float32)
    opt.set("x", x0)
    ropt.set("x", x0.astype(np.float64))
    sig = np.repeat(10.0 ** (-4 + 2 * rng.random(len(sizes))), sizes)
    for t in range(steps):
        g = (rng.standard_normal((n, d)) * sig).astype(np.float32)
        opt.step(g, t, 1e-3)
        ropt.step(g.astype(np.float64), t, 1e-3, rcl)
        if t == warm - 1:
            # warmup LAMB + freeze: fp32 vs fp64 rounding only (measured 5e-7)
            np.testing.assert_allclose(opt.get("v_frozen"), ropt.get("v_frozen"), rtol=1e-5, atol=1e-30)
            xw, xwr = opt.get("x").astype(np.float64), ropt.get("x")
            assert np.linalg.norm(xw - xwr) <= 1e-4 * np.linalg.norm(xwr - x0)
    # Tolerances: norm-wise x drift <= 1e-3 of the distance
    # travelled (measured ~1e-5), momentum <= 1e-5 relative, r within 1e-4.
    x, xr = opt.get("x").astype(np.float64), ropt.get("x")
    assert np.linalg.norm(x - xr) <= 1e-3 * np.linalg.norm(xr - x0)
    m, mr = opt.get("m").astype(np.float64), ropt.get("m")
    assert np.linalg.norm(m - mr) <= 1e-5 * np.linalg.norm(mr)
    np.testing.assert_allclose(opt.scalars()["r_prev"], ropt.scalars()["r_prev"], rtol=1e-4)


def test_ratio_clipping_kat(bl):
    """test_optimizers.cpp:220-256: vf=[4,1], v=[1,1] -> pre 4, r 1.1, c 0.55."""
    hp = bl.HyperParams(total_steps=4, warmup_steps=1, beta1=0.0, beta2=0.0)
    cl = bl.SimCluster(1, 2)
    opt = bl.Optimizer("onebit_lamb", [2], hp, cl)
    opt.set("x", np.array([1.0, 1.0], np.float32))
    opt.step(np.array([[1.0, 1.0]], np.float32), 0, 1e-3)
    assert opt.frozen()
    opt.set("v_frozen", np.array([4.0, 1.0], np.float32))
    opt.set_scalars(c_avg=[0.5], r_prev=[1.0])
    x_before = opt.get("x")
    tr = opt.step(np.array([[1.0, 1.0]], np.float32), 1, 0.01)
    assert tr.v_ratio_preclip[0] == pytest.approx(4.0, rel=1e-12)
    assert tr.r[0] == pytest.approx(1.1, rel=1e-12)
    assert tr.c[0] == pytest.approx(0.55, rel=1e-12)
    x = opt.get("x")
    assert x[0] == pytest.approx(x_before[0] - 0.01 * 0.55 / (2.0 + 1e-6), rel=1e-6)
    assert x[1] == pytest.approx(x_before[1] - 0.01 * 0.55 / (1.0 + 1e-6), rel=1e-6)


def test_scalar_lamb_kat(bl):
    """test_optimizers.cpp:69-93: x' ~ 0.990516, c == c_max."""
    hp = bl.HyperParams(total_steps=10, warmup_steps=0)
    cl = bl.SimCluster(1, 1, compressor="identity")
    opt = bl.Optimizer("lamb", [1], hp, cl)
    opt.set("x", np.array([1.0], np.float32))
    tr = opt.step(np.array([[0.1]], np.float32), 0, 0.01)
    assert tr.c[0] == 0.3
    assert opt.get("x")[0] == pytest.approx(0.990516, rel=1e-5)


def test_warmup_c_avg_closed_form(bl):
    """test_optimizers.cpp:132-177: c_avg = 0.3 (1 - 0.9^t) while c saturates."""
    hp = bl.HyperParams(total_steps=10, warmup_steps=5)
    cl = bl.SimCluster(1, 4)
    opt = bl.Optimizer("onebit_lamb", [4], hp, cl)
    opt.set("x", np.full(4, 1e6, np.float32))
    g = np.array([[0.1, 0.2, -0.1, 0.3]], np.float32)
    for t in range(5):
        tr = opt.step(g, t, 1e-6)
        assert tr.c[0] == 0.3
    assert opt.scalars()["c_avg"][0] == pytest.approx(0.3 * (1 - 0.9 ** 5), rel=1e-14)
    assert opt.frozen()


def test_clip_contracts_and_frozen_variance(bl):
    """test_optimizers.cpp:258-315."""
    hp = bl.HyperParams(total_steps=60, warmup_steps=20)
    cl = bl.SimCluster(2, 9)
    opt = bl.Optimizer("onebit_lamb", [6, 3], hp, cl)
    rng = np.random.default_rng(17)
    prev_r = None
    snap = None
    for t in range(60):
        tr = opt.step(rng.standard_normal((2, 9)).astype(np.float32), t, 5e-3)
        c_avg = opt.scalars()["c_avg"]
        if t < 20:
            assert np.all((tr.c >= 0.01) & (tr.c <= 0.3))
        else:
            assert np.all((tr.r >= 0.5) & (tr.r <= 4.0))
            assert np.all(tr.c >= 0.5 * c_avg - 1e-15) and np.all(tr.c <= 4.0 * c_avg + 1e-15)
            if prev_r is not None:
                assert np.all(np.abs(tr.r / prev_r - 1.0) <= 0.1 + 1e-12)
            prev_r = tr.r
            assert_same(opt.get("v_frozen"), snap)
        if t == 19:
            snap = opt.get("v_frozen")


def test_stage_order_and_gradient_errors(bl):
    """test_optimizers.cpp:637-652."""
    hp = bl.HyperParams(total_steps=10, warmup_steps=0)
    cl = bl.SimCluster(1, 2)
    opt = bl.Optimizer("onebit_lamb", [2], hp, cl)
    with pytest.raises(bl.StageOrderError):
        opt.step(np.array([[1.0, 1.0]], np.float32), 0, 0.01)
    lamb = bl.Optimizer("lamb", [2], hp, cl)
    with pytest.raises(bl.NumericalError, match="non-finite gradient"):
        lamb.step(np.array([[1.0, np.nan]], np.float32), 0, 0.01)
    with pytest.raises(bl.ConfigError):
        bl.Optimizer("lamb", [2], bl.HyperParams(beta1=1.0), cl)


def test_stage_dichotomy_ledger(bl):
    """test_optimizers.cpp:317-346."""
    hp = bl.HyperParams(total_steps=12, warmup_steps=5)
    cl = bl.SimCluster(2, 8)
    opt = bl.Optimizer("onebit_lamb", [8], hp, cl)
    rng = np.random.default_rng(31)
    for t in range(12):
        before = cl.ledger()
        opt.step(rng.standard_normal((2, 8)).astype(np.float32), t, 1e-3)
        after = cl.ledger()
        if t < 5:
            assert after.lossless_bits > before.lossless_bits and after.gather_bits == before.gather_bits
        else:
            assert after.lossless_bits == before.lossless_bits and after.gather_bits > before.gather_bits
    assert cl.ledger().lossless_collectives == 5 and cl.ledger().compressed_collectives == 7


def test_device_resident_step_matches_host_step(bl):
    """Zero-copy device gradients (torch CUDA tensors) == host gradients."""
    import torch

    sizes = [5000, 3, 2048]
    d = sum(sizes)
    res = []
    for dev in (False, True):
        hp = bl.HyperParams(total_steps=8, warmup_steps=3)
        cl = bl.SimCluster(2, d)
        opt = bl.Optimizer("onebit_lamb", sizes, hp, cl)
        rng = np.random.default_rng(9)
        for t in range(8):
            g = (rng.standard_normal((2, d)) * 1e-3).astype(np.float32)
            opt.step(torch.from_numpy(g).cuda() if dev else g, t, 1e-3, trace=t == 7)
        res.append(opt.get("x"))
    assert_same(res[0], res[1])


@pytest.mark.parametrize("lead", [1, 2, 3])
@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("variant", ["onebit_lamb", "lamb_basic_1bit", "lamb"])
def test_misaligned_layer_full_tiles_bitexact(bl, lead, n, variant):
    """A layer of full tiles starting 1-3 floats past a 16-byte boundary takes
    the kernels' misaligned full-tile path (W1/W2/K5/K6); bit-exact with the
    f32 oracle like the aligned and per-row paths."""
    run_pair(bl, [lead, 3 * 4096 + 5, 7, 4096], n, steps=8, warmup=3, seed=40 + lead, variant=variant)
