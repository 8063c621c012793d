"""CPU suite: pin the oracle (oracle/bitlamb_oracle.c) before trusting it.

1. Golden fixtures produced by the reference library itself
   (tests/golden/make_golden.py): the f64 build must reproduce them
   bit-for-bit, the f32 build within fp32 tolerance.
2. The reference's own known-answer tests (test_compression.cpp,
   test_comm_sim.cpp, test_fusion.cpp, test_optimizers.cpp) on both builds.
3. When oracle/_ref is built (development container), randomized
   differential runs f64-oracle == reference, bit-exact, all five variants.
4. The canonical tile-tree reduction order of the f32 build, restated in numpy.
"""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from oracle import oracle as O

from conftest import have_ref

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


def load(path):
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


# ---------------------------------------------------------------------------
# 1. golden fixtures from the reference
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("path", [p for p in GOLDEN if "collective" in p], ids=os.path.basename)
@pytest.mark.parametrize("which", ["f64", "f32"])
def test_golden_collective(path, which):
    g = load(path)
    n, d, calls = int(g["n"]), int(g["d"]), int(g["calls"])
    c = O.Cluster(which, n, d)
    for k in range(calls):
        out = c.compressed_allreduce(g[f"in{k}"], float(g[f"es{k}"]))
        pk = np.stack([np.frombuffer(c.packet(i, j), np.uint8) for i in range(n) for j in range(n)])
        werr = np.stack([c.worker_error(i) for i in range(n)])
        serr = np.stack([c.server_error(j) for j in range(n)])
        if which == "f64":
            np.testing.assert_array_equal(out, g[f"out{k}"])
            np.testing.assert_array_equal(werr, g[f"werr{k}"])
            np.testing.assert_array_equal(serr, g[f"serr{k}"])
            np.testing.assert_array_equal(pk, g[f"pkt{k}"])
        else:
            nb = (c.chunk + 7) // 8
            if k == 0:  # identical inputs, zero residuals: signs bit-exact
                np.testing.assert_array_equal(pk[:, :nb], g[f"pkt{k}"][:, :nb])
            np.testing.assert_allclose(out, g[f"out{k}"], rtol=1e-5, atol=1e-6)
            np.testing.assert_allclose(werr, g[f"werr{k}"], rtol=1e-4, atol=1e-5)
    led = c.ledger()
    assert [led[k] for k in ("gather_bits", "scatter_bits", "lossless_bits", "baseline_equivalent_bits",
                             "compressed_collectives", "lossless_collectives")] == list(g["ledger"])
    if which == "f64":
        np.testing.assert_array_equal(c.stats(), g["stats"])


@pytest.mark.parametrize("path", [p for p in GOLDEN if "optimizer" in p], ids=os.path.basename)
@pytest.mark.parametrize("which", ["f64", "f32"])
def test_golden_optimizer(path, which):
    g = load(path)
    sizes = [int(s) for s in g["sizes"]]
    n, steps, warm = int(g["n"]), int(g["steps"]), int(g["warmup"])
    hp = O.HyperParams(total_steps=steps, warmup_steps=warm, weight_decay=float(g["wd"]),
                       scaled_error_feedback=bool(g["scaled"]))
    opt = O.Optimizer(which, str(g["variant"]), sizes, hp)
    cl = O.Cluster(which, n, sum(sizes))
    opt.set("x", g["x0"])
    for t in range(steps):
        tr = opt.step(g[f"g{t}"], t, 1e-3, cl)
        got = np.stack([tr["c"], tr["r"], tr["v_norm"], tr["v_ratio_preclip"]])
        if which == "f64":
            np.testing.assert_array_equal(got, g[f"trace{t}"])
        else:
            np.testing.assert_allclose(got, g[f"trace{t}"], rtol=1e-4)
    for k in ("x", "m", "v", "v_frozen", "m_prev"):
        if which == "f64":
            np.testing.assert_array_equal(opt.get(k), g[k], err_msg=k)
        else:
            ref = g[k]
            scale = max(np.abs(ref).max(), 1e-30)
            assert np.abs(opt.get(k) - ref).max() <= 1e-4 * scale, k
    sc = opt.scalars()
    if which == "f64":
        np.testing.assert_array_equal(sc["c_avg"], g["c_avg"])
        np.testing.assert_array_equal(sc["r_prev"], g["r_prev"])
        np.testing.assert_array_equal(sc["scale_coeff"], g["coeff"])


# ---------------------------------------------------------------------------
# 2. the reference's own known-answer tests
# ---------------------------------------------------------------------------
BOTH = pytest.mark.parametrize("which", ["f64", "f32"])


@BOTH
def test_kat_compress_signs_and_scale(which):
    """test_compression.cpp:47-57."""
    b, s, dec, dl = O.compress_with_feedback(which, [2.0, -1.0, 0.5, -0.5], [0, 0, 0, 0])
    assert s == 1.0 and b[0] & 0xF == 0b0101
    np.testing.assert_array_equal(dec, [1.0, -1.0, 1.0, -1.0])


@BOTH
def test_kat_zero_and_constant(which):
    """test_compression.cpp:59-76."""
    b, s, dec, _ = O.compress_with_feedback(which, [0, 0, 0], [0, 0, 0])
    assert s == 0.0 and not dec.any()
    _, s, dec, _ = O.compress_with_feedback(which, [0.75, 0.75, -0.75], [0, 0, 0])
    np.testing.assert_array_equal(dec, [0.75, 0.75, -0.75])
    _, s, dec, _ = O.compress_with_feedback(which, [1.0, -3.0], [0, 0])
    assert s == 2.0


@BOTH
def test_kat_nonfinite_rejected(which):
    """test_compression.cpp:78-82."""
    with pytest.raises(O.OracleError) as e:
        O.compress_with_feedback(which, [1.0, np.nan], [0, 0])
    assert e.value.kind == "InvalidArgument"


@BOTH
def test_kat_feedback_split(which):
    """test_compression.cpp:84-100."""
    _, _, dec, dl = O.compress_with_feedback(which, [0.3], [0])
    assert dec[0] == O.lib(which).real(0.3) and dl[0] == 0.0
    _, _, dec, dl = O.compress_with_feedback(which, [1.0, 0.0], [0, 0])
    np.testing.assert_array_equal(dec, [0.5, 0.5])
    np.testing.assert_array_equal(dl, [0.5, -0.5])


@BOTH
def test_kat_identity_kills_residual(which):
    """test_compression.cpp:102-112."""
    rng = np.random.default_rng(1)
    dl = np.zeros(8)
    for _ in range(20):
        v = rng.standard_normal(8).astype(np.float32)
        _, _, dec, dl = O.compress_with_feedback(which, v, dl, kind="identity")
        np.testing.assert_array_equal(dec, v.astype(O.lib(which).real))
        assert not dl.any()


@BOTH
def test_kat_compensation_identity_and_bounds(which):
    """test_compression.cpp:114-160 (tolerance per precision)."""
    tol = 1e-12 if which == "f64" else 2.0 ** -23
    for d in (1, 2, 17, 256):
        dl = np.zeros(d, O.lib(which).real)
        mx_d = mx_c = 0.0
        for step in range(100):
            v = np.random.default_rng(7000 + step + d).standard_normal(d).astype(np.float32)
            corr = v.astype(np.float64) + dl
            _, _, dec, dl = O.compress_with_feedback(which, v, dl)
            lhs, rhs = corr, dec.astype(np.float64) + dl
            den = np.maximum(np.maximum(np.abs(lhs), np.abs(dec)), 1e-300)
            assert np.all(np.abs(lhs - rhs) <= tol * den)
            assert np.all((corr <= 0) | (dec >= 0)) and np.all((corr >= 0) | (dec <= 0))
            mx_c = max(mx_c, np.abs(corr).max())
            mx_d = max(mx_d, np.abs(dl).max())
        assert mx_d <= 2 * mx_c


@BOTH
def test_kat_wire_layout(which):
    """test_compression.cpp:169-191: golden bytes b9 02 00 00 80 3f."""
    v = [1.0, -1.0, -1.0, 1.0, 1.0, 1.0, -1.0, 1.0, -1.0, 1.0]
    b, _, _, _ = O.compress_with_feedback(which, v, [0.0] * 10)
    assert b == bytes([0b10111001, 0b00000010, 0x00, 0x00, 0x80, 0x3F])


@BOTH
def test_kat_volume_reduction(which):
    """test_comm_sim.cpp:39-51."""
    assert abs(O.volume_reduction(which, 0.167, 16, 1.0) - 4.56) <= 0.05
    assert abs(O.volume_reduction(which, 0.193, 16, 1.0) - 4.11) <= 0.05
    assert O.volume_reduction(which, 1.0, 16, 1.0) == 1.0
    with pytest.raises(O.OracleError):
        O.volume_reduction(which, -0.1, 16, 1.0)


@BOTH
def test_kat_lossless_and_identity_collapse(which):
    """test_comm_sim.cpp:53-134."""
    c = O.Cluster(which, 2, 2, kind="identity")
    np.testing.assert_array_equal(c.lossless_allreduce([[1, 2], [3, 4]]), [2, 3])
    for n in (1, 2, 3, 4, 8):
        for d in (1, 5, 16, 37):
            x = np.random.default_rng(1000 + n * 100 + d).standard_normal((n, d)).astype(np.float32)
            a = O.Cluster(which, n, d, kind="identity").compressed_allreduce(x)
            b = O.Cluster(which, n, d, kind="identity").lossless_allreduce(x)
            np.testing.assert_array_equal(a, b)


def test_kat_two_worker_scripted_f64():
    """test_comm_sim.cpp:163-222 (fp64, exact ==)."""
    n, d, ch = 2, 4, 2
    x = np.random.default_rng(4242).standard_normal((n, d))
    c = O.Cluster("f64", n, d)
    out = c.compressed_allreduce(x)
    wd = np.zeros((n, d))
    sd = np.zeros((n, ch))
    sent = {}
    for i in range(n):
        for j in range(n):
            corr = x[i, j * ch:(j + 1) * ch] + wd[i, j * ch:(j + 1) * ch]
            s = np.abs(corr).sum() / ch
            dec = np.where(corr >= 0, s, -s)
            wd[i, j * ch:(j + 1) * ch] = corr - dec
            sent[i, j] = dec
    exp = np.zeros(d)
    for j in range(n):
        avg = (sent[0, j] + sent[1, j]) / n
        corr = avg + sd[j]
        s = np.abs(corr).sum() / ch
        dec = np.where(corr >= 0, s, -s)
        sd[j] = corr - dec
        exp[j * ch:(j + 1) * ch] = dec
    np.testing.assert_array_equal(out, exp)
    for i in range(n):
        np.testing.assert_array_equal(c.worker_error(i), wd[i])
        np.testing.assert_array_equal(c.server_error(i), sd[i])


@BOTH
def test_kat_ledger_padding(which):
    """test_comm_sim.cpp:239-259."""
    c = O.Cluster(which, 2, 5)
    out = c.compressed_allreduce(np.random.default_rng(333).standard_normal((2, 5)))
    assert out.shape == (5,)
    led = c.ledger()
    assert led["gather_bits"] == 35 + 34 == led["scatter_bits"]
    assert led["baseline_equivalent_bits"] == 2 * 5 * 16 and led["compressed_collectives"] == 1


@BOTH
def test_kat_pad_carries_error(which):
    """SURVEY Appendix C pad probe: d=5, n=2 -> werr[0] = [-1, 0, 1, -1, 2, -3]."""
    c = O.Cluster(which, 2, 5)
    c.compressed_allreduce([[1, -2, 3, -4, 5], [0.5] * 5])
    np.testing.assert_array_equal(c.worker_error(0), [-1, 0, 1, -1, 2, -3])


@BOTH
def test_kat_scalar_lamb(which):
    """test_optimizers.cpp:69-93."""
    opt = O.Optimizer(which, "lamb", [1], O.HyperParams(total_steps=10))
    opt.set("x", [1.0])
    tr = opt.step([[0.1]], 0, 0.01, O.Cluster(which, 1, 1, kind="identity"))
    assert tr["c"][0] == 0.3
    assert opt.get("x")[0] == pytest.approx(0.990516, rel=1e-5)


@BOTH
def test_kat_zero_norm_rule(which):
    """test_optimizers.cpp:95-130."""
    hp = O.HyperParams(total_steps=4)
    opt = O.Optimizer(which, "lamb", [3], hp)
    opt.set("x", [1.0, -2.0, 0.5])
    tr = opt.step(np.zeros((1, 3)), 0, 0.01, O.Cluster(which, 1, 3, kind="identity"))
    assert tr["c"][0] == 0.3
    np.testing.assert_array_equal(opt.get("x"), np.array([1.0, -2.0, 0.5], O.lib(which).real))
    z = O.Optimizer(which, "lamb", [3], hp)
    tr = z.step(np.zeros((1, 3)), 0, 0.01, O.Cluster(which, 1, 3, kind="identity"))
    assert tr["c"][0] == 0.3  # clip(1, 0.01, 0.3)


@BOTH
def test_kat_c_avg_closed_form(which):
    """test_optimizers.cpp:132-177."""
    opt = O.Optimizer(which, "onebit_lamb", [4], O.HyperParams(total_steps=10, warmup_steps=5))
    opt.set("x", [1e6] * 4)
    cl = O.Cluster(which, 1, 4, kind="identity")
    for t in range(5):
        assert opt.step([[0.1, 0.2, -0.1, 0.3]], t, 1e-6, cl)["c"][0] == 0.3
    assert opt.scalars()["c_avg"][0] == pytest.approx(0.3 * (1 - 0.9 ** 5), rel=1e-14)
    assert opt.frozen


@BOTH
def test_kat_ratio_clipping(which):
    """test_optimizers.cpp:220-256."""
    hp = O.HyperParams(total_steps=4, warmup_steps=1, beta1=0.0, beta2=0.0)
    opt = O.Optimizer(which, "onebit_lamb", [2], hp)
    opt.set("x", [1.0, 1.0])
    cl = O.Cluster(which, 1, 2, kind="identity")
    opt.step([[1.0, 1.0]], 0, 1e-3, cl)
    opt.set("v_frozen", [4.0, 1.0])
    opt.set_scalars([0.5], [1.0])
    xb = opt.get("x").astype(np.float64)
    tr = opt.step([[1.0, 1.0]], 1, 0.01, cl)
    assert tr["v_ratio_preclip"][0] == pytest.approx(4.0, rel=1e-12)
    assert tr["r"][0] == pytest.approx(1.1, rel=1e-12)
    assert tr["c"][0] == pytest.approx(0.55, rel=1e-12)
    rel = 1e-12 if which == "f64" else 1e-6
    assert opt.get("x")[0] == pytest.approx(xb[0] - 0.01 * 0.55 / (2.0 + 1e-6), rel=rel)


@BOTH
def test_kat_momentum_scales(which):
    """test_fusion.cpp:90-100 via finalize_warmup: magnitudes 0.1 / 0.4 ->
    coefficients 2.5 / 0.625 (beta1 = 0 makes m the last gradient)."""
    hp = O.HyperParams(total_steps=2, warmup_steps=1, beta1=0.0)
    opt = O.Optimizer(which, "onebit_lamb", [4, 2], hp)
    opt.step([[0.1, -0.1, 0.1, -0.1, 0.4, -0.4]], 0, 1e-3, O.Cluster(which, 1, 6, kind="identity"))
    co = opt.scalars()["scale_coeff"]
    assert co[0] == pytest.approx(2.5, rel=1e-6) and co[1] == pytest.approx(0.625, rel=1e-6)


@BOTH
def test_kat_errors(which):
    """test_optimizers.cpp:34-51, 637-652."""
    with pytest.raises(O.OracleError) as e:
        O.Optimizer(which, "lamb", [2], O.HyperParams(beta1=1.0))
    assert e.value.kind == "ConfigError"
    with pytest.raises(O.OracleError) as e:
        O.Optimizer(which, "lamb", [2], O.HyperParams(total_steps=10, warmup_steps=20))
    assert e.value.kind == "ConfigError"
    opt = O.Optimizer(which, "onebit_lamb", [2], O.HyperParams(total_steps=10))
    with pytest.raises(O.OracleError) as e:
        opt.step([[1.0, 1.0]], 0, 0.01, O.Cluster(which, 1, 2))
    assert e.value.kind == "StageOrderError"
    lamb = O.Optimizer(which, "lamb", [2], O.HyperParams(total_steps=10))
    with pytest.raises(O.OracleError) as e:
        lamb.step([[1.0, np.nan]], 0, 0.01, O.Cluster(which, 1, 2))
    assert e.value.kind == "RuntimeError"


# ---------------------------------------------------------------------------
# 3. differential: f64 oracle == reference library (bit-exact)
# ---------------------------------------------------------------------------
needs_ref = pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("n,d", [(1, 6), (2, 5), (3, 10), (4, 23), (8, 37), (4, 10000), (2, 20001)])
def test_f64_oracle_equals_reference_collective(n, d):
    rng = np.random.default_rng(n * 1000 + d)
    a, b = O.Cluster("ref", n, d), O.Cluster("f64", n, d)
    for step in range(4):
        x = rng.standard_normal((n, d))
        es = 1.0 if step < 3 else 0.8
        np.testing.assert_array_equal(a.compressed_allreduce(x, es), b.compressed_allreduce(x, es))
        for i in range(n):
            np.testing.assert_array_equal(a.worker_error(i), b.worker_error(i))
            np.testing.assert_array_equal(a.server_error(i), b.server_error(i))
            for j in range(n):
                assert a.packet(i, j) == b.packet(i, j)
    assert a.ledger() == b.ledger()
    np.testing.assert_array_equal(a.stats(), b.stats())


@needs_ref
@pytest.mark.parametrize("variant", ["lamb", "adam", "onebit_lamb", "lamb_basic_1bit", "onebit_adam"])
def test_f64_oracle_equals_reference_optimizer(variant):
    sizes = [3000, 2, 1024, 1023, 5000, 3]
    d = sum(sizes)
    rng = np.random.default_rng(11)
    for n, wd, scaled in ((1, 0.0, False), (4, 0.01, True)):
        hp = O.HyperParams(total_steps=25, warmup_steps=8, weight_decay=wd, scaled_error_feedback=scaled)
        a, b = O.Optimizer("ref", variant, sizes, hp), O.Optimizer("f64", variant, sizes, hp)
        x0 = rng.standard_normal(d) * 0.02
        a.set("x", x0)
        b.set("x", x0)
        ca, cb = O.Cluster("ref", n, d), O.Cluster("f64", n, d)
        for t in range(25):
            g = rng.standard_normal((n, d)) * 1e-2
            ta, tb = a.step(g, t, 1e-3, ca), b.step(g, t, 1e-3, cb)
            for k in ("c", "r", "v_norm", "v_ratio_preclip", "compressed"):
                np.testing.assert_array_equal(ta[k], tb[k])
        for k in ("x", "m", "v", "v_frozen", "m_prev"):
            np.testing.assert_array_equal(a.get(k), b.get(k))


@needs_ref
def test_f64_oracle_matches_reference_errors():
    for w in ("ref", "f64"):
        c = O.Cluster(w, 2, 4)
        with pytest.raises(O.OracleError) as e:
            c.compressed_allreduce(np.zeros((1, 4)))
        assert e.value.kind == "DimensionError"
        with pytest.raises(O.OracleError) as e:
            O.Cluster(w, 0, 4)
        assert e.value.kind == "InvalidArgument"


# ---------------------------------------------------------------------------
# 4. the canonical tile-tree order of the f32 build
# ---------------------------------------------------------------------------
def numpy_tile_tree(x: np.ndarray, square: bool) -> float:
    x = x.astype(np.float64)
    x = x * x if square else np.abs(x)
    T = -(-x.size // 4096)
    xp = np.zeros(T * 4096)
    xp[: x.size] = x
    tiles = xp.reshape(T, 32, 32, 4)  # tile, row, lane, element

    def bfly(a):
        a = a.copy()
        for s in (16, 8, 4, 2, 1):
            a = a + a[..., np.arange(32) ^ s]
        return a[..., 0]

    lane = np.zeros((T, 32))
    for r in range(32):
        for q in range(4):
            lane = lane + tiles[:, r, :, q]
    part = bfly(lane)
    stripe = np.zeros(1024)
    for t in range(T):
        stripe[t % 1024] += part[t]
    return float(bfly(bfly(stripe.reshape(32, 32))[None, :])[0])


@pytest.mark.parametrize("n", [1, 5, 4096, 4097, 100_003, 5_000_000])
def test_f32_reduction_order_is_the_tile_tree(n):
    x = np.random.default_rng(n).standard_normal(n).astype(np.float32) * \
        np.float32(10.0) ** np.random.default_rng(n + 1).integers(-6, 6, n).astype(np.float32)
    for kind in (0, 1):
        assert O.canonical_sum("f32", x, kind) == numpy_tile_tree(x, kind == 1)
    # and it is a faithful sum (fp64 accumulation): within 1e-13 of the exact sum
    exact = float(np.sum(np.abs(x.astype(np.float64))))
    assert abs(O.canonical_sum("f32", x, 0) - exact) <= 1e-13 * exact
