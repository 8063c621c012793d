"""Generate golden fixtures by running the REFERENCE library itself.

Runs oracle/_ref/libbitlamb_ref.so (the unmodified reference sources in
/root/reference/proj/src compiled by oracle/Makefile, driven through
oracle/ref_shim.cpp) on small seeded cases and stores inputs and outputs as
.npz files next to this script.  The fixtures travel with the repo so the
CPU suite can pin the oracle restatement without /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def f32(a):
    """fp32-representable fp64 values (identical inputs for every checker)."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def collective_case(n: int, d: int, calls: int, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    c = O.Cluster("ref", n, d)
    out = {"n": n, "d": d, "calls": calls}
    for k in range(calls):
        x = f32(rng.standard_normal((n, d)))
        es = 1.0 if k < calls - 1 else 0.5
        out[f"in{k}"] = x
        out[f"es{k}"] = es
        out[f"out{k}"] = c.compressed_allreduce(x, es)
        out[f"werr{k}"] = np.stack([c.worker_error(i) for i in range(n)])
        out[f"serr{k}"] = np.stack([c.server_error(j) for j in range(n)])
        out[f"pkt{k}"] = np.stack([np.frombuffer(c.packet(i, j), np.uint8)
                                   for i in range(n) for j in range(n)])
    led = c.ledger()
    out["ledger"] = np.array([led[k] for k in ("gather_bits", "scatter_bits", "lossless_bits",
                                               "baseline_equivalent_bits", "compressed_collectives",
                                               "lossless_collectives")], dtype=np.uint64)
    out["stats"] = c.stats()
    return out


def optimizer_case(variant: str, sizes, n: int, steps: int, warmup: int, seed: int, wd: float = 0.0,
                   scaled: bool = False) -> dict:
    rng = np.random.default_rng(seed)
    d = sum(sizes)
    hp = O.HyperParams(total_steps=steps, warmup_steps=warmup, weight_decay=wd,
                       scaled_error_feedback=scaled)
    opt = O.Optimizer("ref", variant, sizes, hp)
    cl = O.Cluster("ref", n, d)
    x0 = f32(rng.standard_normal(d) * 0.02)
    opt.set("x", x0)
    sig = np.repeat(10.0 ** (-4 + 2 * rng.random(len(sizes))), sizes)
    out = {"variant": variant, "sizes": np.asarray(sizes), "n": n, "steps": steps, "warmup": warmup,
           "wd": wd, "scaled": scaled, "x0": x0}
    for t in range(steps):
        g = f32(rng.standard_normal((n, d)) * sig)
        out[f"g{t}"] = g
        tr = opt.step(g, t, 1e-3, cl)
        out[f"trace{t}"] = np.stack([tr["c"], tr["r"], tr["v_norm"], tr["v_ratio_preclip"]])
    for k in ("x", "m", "v", "v_frozen", "m_prev"):
        out[k] = opt.get(k)
    sc = opt.scalars()
    out["c_avg"], out["r_prev"], out["coeff"] = sc["c_avg"], sc["r_prev"], sc["scale_coeff"]
    return out


def main():
    cases = {
        "collective_n2_d5": collective_case(2, 5, 3, 1),
        "collective_n4_d37": collective_case(4, 37, 3, 2),
        "collective_n3_d4099": collective_case(3, 4099, 3, 3),
        "collective_n8_d9000": collective_case(8, 9000, 2, 4),
        "optimizer_onebit_lamb_n2": optimizer_case("onebit_lamb", [300, 2, 1024, 5], 2, 14, 4, 5),
        "optimizer_onebit_lamb_n4_wd": optimizer_case("onebit_lamb", [4100, 3, 17], 4, 10, 3, 6,
                                                      wd=0.01, scaled=True),
        "optimizer_lamb_n1": optimizer_case("lamb", [64, 7], 1, 6, 0, 7),
    }
    for name, data in cases.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
        print("wrote", name)


if __name__ == "__main__":
    main()
