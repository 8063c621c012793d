"""ctypes face of the parity checkers — TEST INFRASTRUCTURE ONLY.

Loads any of the three checker libraries behind the common ``oc_*`` C API:

* ``ref``  — oracle/_ref/libbitlamb_ref.so: the UNMODIFIED reference library
  (/root/reference/proj/src) plus oracle/ref_shim.cpp; fp64.
* ``f64``  — oracle/liboracle_f64.so: the C restatement, fp64, reference order.
* ``f32``  — oracle/liboracle_f32.so: the C restatement, fp32, tile-tree order
  (the bit-exact target of the B200 kernels).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference legs import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "ref": os.path.join(HERE, "_ref", "libbitlamb_ref.so"),
    "f64": os.path.join(HERE, "liboracle_f64.so"),
    "f32": os.path.join(HERE, "liboracle_f32.so"),
}

# bl_status / oc status codes -> Python exception names (errors.hpp:26-53)
STATUS = {
    1: "DimensionError",
    2: "StageOrderError",
    3: "ConfigError",
    4: "InvalidArgument",
    5: "RuntimeError",
    6: "LogicError",
    7: "Other",
}

VARIANTS = {"lamb": 0, "adam": 1, "onebit_lamb": 2, "lamb_basic_1bit": 3, "onebit_adam": 4}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, str(code))
        self.msg = msg


@dataclass
class HyperParams:
    """Mirror of bitlamb::HyperParams (optimizers.hpp:45-64), paper defaults."""

    beta1: float = 0.9
    beta2: float = 0.999
    beta3: float = 0.9
    eta: float = 1e-6
    c_min: float = 0.01
    c_max: float = 0.3
    r_min: float = 0.5
    r_max: float = 4.0
    r_threshold: float = 0.1
    weight_decay: float = 0.0
    division_floor: float = 1e-12
    total_steps: int = 0
    warmup_steps: int = 0
    scaled_error_feedback: bool = False

    def doubles(self) -> list[float]:
        return [self.beta1, self.beta2, self.beta3, self.eta, self.c_min, self.c_max,
                self.r_min, self.r_max, self.r_threshold, self.weight_decay,
                self.division_floor]


_LIBS: dict[str, "Lib"] = {}


class Lib:
    def __init__(self, which: str):
        path = PATHS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"checker library {path} not built (run `make -C oracle`)")
        self.which = which
        self.so = C.CDLL(path)
        so = self.so
        so.oc_last_error.restype = C.c_char_p
        so.oc_real_bytes.restype = C.c_int
        self.real = np.float64 if so.oc_real_bytes() == 8 else np.float32
        P = C.c_void_p
        u64 = C.c_uint64
        so.oc_cluster_new.argtypes = [C.c_int, u64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        so.oc_cluster_free.argtypes = [P]
        so.oc_cluster_padded.argtypes = [P]
        so.oc_cluster_padded.restype = u64
        so.oc_cluster_chunk.argtypes = [P]
        so.oc_cluster_chunk.restype = u64
        so.oc_cluster_compressed_allreduce_n.argtypes = [P, P, C.c_int, u64, C.c_double, P]
        so.oc_cluster_lossless_allreduce.argtypes = [P, P, P]
        so.oc_cluster_worker_error.argtypes = [P, C.c_int, P]
        so.oc_cluster_server_error.argtypes = [P, C.c_int, P]
        so.oc_cluster_ledger.argtypes = [P, P]
        so.oc_cluster_stats.argtypes = [P, P]
        so.oc_cluster_compensation_checks.argtypes = [P]
        so.oc_cluster_compensation_checks.restype = u64
        so.oc_cluster_packet.argtypes = [P, C.c_int, C.c_int, P]
        so.oc_compress_with_feedback.argtypes = [P, P, u64, C.c_int, C.c_double, P, P, P]
        so.oc_volume_reduction.argtypes = [C.c_double, C.c_double, C.c_double, P]
        so.oc_opt_new.argtypes = [C.c_int, P, C.c_int, P, u64, u64, C.c_int, C.POINTER(C.c_void_p)]
        so.oc_opt_free.argtypes = [P]
        so.oc_opt_step.argtypes = [P, P, P, C.c_int, u64, C.c_double, P, P]
        so.oc_opt_get.argtypes = [P, C.c_int, P]
        so.oc_opt_set.argtypes = [P, C.c_int, P]
        so.oc_opt_get_scalars.argtypes = [P, P]
        so.oc_opt_set_scalars.argtypes = [P, P]
        so.oc_opt_frozen.argtypes = [P]
        if which == "ref":
            so.oc_set_threads.argtypes = [C.c_int]
            so.oc_set_threads.restype = C.c_int
            so.oc_opt_load_grads.argtypes = [P, P, C.c_int]
            so.oc_opt_step_loaded.argtypes = [P, P, u64, C.c_double, P, P]
        if which != "ref":
            so.oc_cluster_set_tolerance.argtypes = [P, C.c_double]
            so.oc_cluster_server_packet.argtypes = [P, C.c_int, P]
            so.oc_worker_compress.argtypes = [P, u64, C.c_int, P, C.c_double, P]
            so.oc_server_reduce.argtypes = [P, u64, C.c_int, P, C.c_double, P]
            so.oc_decompress.argtypes = [P, u64, P]
            so.oc_canonical_sum.argtypes = [P, u64, C.c_int]
            so.oc_canonical_sum.restype = C.c_double

    def check(self, st: int) -> None:
        if st != 0:
            raise OracleError(st, self.so.oc_last_error().decode())

    def arr(self, a) -> np.ndarray:
        return np.ascontiguousarray(a, dtype=self.real)


def set_reference_threads(n: int) -> int:
    """OpenMP threads used by the reference library; returns the team size."""
    return int(lib("ref").so.oc_set_threads(int(n)))


def lib(which: str) -> Lib:
    if which not in _LIBS:
        _LIBS[which] = Lib(which)
    return _LIBS[which]


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Cluster:
    """SimCluster (comm_sim.hpp:72-148) on one of the checker libraries."""

    def __init__(self, which: str, n: int, dim: int, kind: str = "onebit",
                 baseline_bits: int = 16, verify: bool = False, tol: float | None = None):
        self.L = lib(which)
        h = C.c_void_p()
        self.L.check(self.L.so.oc_cluster_new(n, dim, 0 if kind == "onebit" else 1,
                                              baseline_bits, int(verify), C.byref(h)))
        self.h = h
        self.n, self.dim = n, dim
        if tol is not None and which != "ref":
            self.L.so.oc_cluster_set_tolerance(self.h, tol)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.so.oc_cluster_free(self.h)
            self.h = None

    @property
    def padded(self) -> int:
        return int(self.L.so.oc_cluster_padded(self.h))

    @property
    def chunk(self) -> int:
        return int(self.L.so.oc_cluster_chunk(self.h))

    def compressed_allreduce(self, inputs, error_scale: float = 1.0) -> np.ndarray:
        x = self.L.arr(inputs)
        n_in = x.shape[0] if x.ndim == 2 else 1
        length = x.shape[-1]
        out = np.zeros(max(self.dim, length), dtype=self.L.real)
        self.L.check(self.L.so.oc_cluster_compressed_allreduce_n(
            self.h, ptr(x), n_in, length, error_scale, ptr(out)))
        return out[: self.dim]

    def lossless_allreduce(self, inputs) -> np.ndarray:
        x = self.L.arr(inputs)
        assert x.shape == (self.n, self.dim)
        out = np.zeros(self.dim, dtype=self.L.real)
        self.L.check(self.L.so.oc_cluster_lossless_allreduce(self.h, ptr(x), ptr(out)))
        return out

    def worker_error(self, i: int) -> np.ndarray:
        out = np.zeros(self.padded, dtype=self.L.real)
        self.L.so.oc_cluster_worker_error(self.h, i, ptr(out))
        return out

    def server_error(self, j: int) -> np.ndarray:
        out = np.zeros(self.chunk, dtype=self.L.real)
        self.L.so.oc_cluster_server_error(self.h, j, ptr(out))
        return out

    def ledger(self) -> dict:
        out = np.zeros(6, dtype=np.uint64)
        self.L.so.oc_cluster_ledger(self.h, ptr(out))
        keys = ["gather_bits", "scatter_bits", "lossless_bits", "baseline_equivalent_bits",
                "compressed_collectives", "lossless_collectives"]
        return {k: int(v) for k, v in zip(keys, out)}

    def stats(self) -> np.ndarray:
        out = np.zeros(2 * self.n * 5, dtype=np.float64)
        self.L.so.oc_cluster_stats(self.h, ptr(out))
        return out.reshape(2, self.n, 5)

    def compensation_checks(self) -> int:
        return int(self.L.so.oc_cluster_compensation_checks(self.h))

    def packet(self, worker: int, server: int) -> bytes:
        out = np.zeros((self.chunk + 7) // 8 + 4, dtype=np.uint8)
        self.L.check(self.L.so.oc_cluster_packet(self.h, worker, server, ptr(out)))
        return out.tobytes()

    def server_packet(self, server: int) -> bytes:
        out = np.zeros((self.chunk + 7) // 8 + 4, dtype=np.uint8)
        self.L.check(self.L.so.oc_cluster_server_packet(self.h, server, ptr(out)))
        return out.tobytes()


def compress_with_feedback(which: str, v, delta, kind: str = "onebit", error_scale: float = 1.0):
    """compression.hpp:106-118; returns (wire_bytes, scale, decompressed, new_delta)."""
    L = lib(which)
    v = L.arr(v)
    dl = L.arr(delta).copy()
    d = v.shape[0]
    out = np.zeros(max(1, (d + 7) // 8 + 4), dtype=np.uint8)
    dec = np.zeros(max(d, 1), dtype=L.real)
    sc = C.c_double()
    L.check(L.so.oc_compress_with_feedback(ptr(v), ptr(dl), d, 0 if kind == "onebit" else 1,
                                           error_scale, ptr(out), C.addressof(sc), ptr(dec)))
    return out[: (d + 7) // 8 + 4].tobytes(), sc.value, dec[:d], dl


def volume_reduction(which: str, w: float, bb: float, cb: float) -> float:
    L = lib(which)
    out = C.c_double()
    L.check(L.so.oc_volume_reduction(w, bb, cb, C.addressof(out)))
    return out.value


def canonical_sum(which: str, x, kind: int) -> float:
    L = lib(which)
    a = L.arr(x)
    return float(L.so.oc_canonical_sum(ptr(a), a.shape[0], kind))


class Optimizer:
    """bitlamb::Optimizer (optimizers.hpp:93-145) on a checker library."""

    WHICH = {"x": 0, "m": 1, "v": 2, "v_frozen": 3, "m_prev": 4}

    def __init__(self, which: str, variant: str, sizes, hp: HyperParams):
        self.L = lib(which)
        self.sizes = [int(s) for s in sizes]
        self.d = sum(self.sizes)
        sz = np.asarray(self.sizes, dtype=np.uint64)
        hpd = np.asarray(hp.doubles(), dtype=np.float64)
        h = C.c_void_p()
        self.L.check(self.L.so.oc_opt_new(VARIANTS[variant], ptr(sz), len(self.sizes), ptr(hpd),
                                          hp.total_steps, hp.warmup_steps,
                                          int(hp.scaled_error_feedback), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.so.oc_opt_free(self.h)
            self.h = None

    def step(self, grads, t: int, lr: float, cluster: Cluster) -> dict:
        g = self.L.arr(grads)
        n = g.shape[0]
        Ln = len(self.sizes)
        tr = np.zeros(4 * Ln, dtype=np.float64)
        comp = C.c_int()
        self.L.check(self.L.so.oc_opt_step(self.h, cluster.h, ptr(g), n, t, lr, ptr(tr),
                                           C.addressof(comp)))
        return {"c": tr[:Ln].copy(), "r": tr[Ln:2 * Ln].copy(), "v_norm": tr[2 * Ln:3 * Ln].copy(),
                "v_ratio_preclip": tr[3 * Ln:].copy(), "compressed": bool(comp.value)}

    def load_grads(self, grads) -> None:
        """ref only: convert the n fused gradients once (bench reference arm)."""
        g = self.L.arr(grads)
        self.L.check(self.L.so.oc_opt_load_grads(self.h, ptr(g), g.shape[0]))

    def step_loaded(self, t: int, lr: float, cluster: Cluster) -> tuple[float, bool]:
        """ref only: the stock Optimizer::step on the loaded gradients; returns
        (seconds measured around the call in C++, compressed)."""
        sec = C.c_double()
        comp = C.c_int()
        self.L.check(self.L.so.oc_opt_step_loaded(self.h, cluster.h, t, lr, C.addressof(sec),
                                                  C.addressof(comp)))
        return sec.value, bool(comp.value)

    def get(self, name: str) -> np.ndarray:
        out = np.zeros(self.d, dtype=self.L.real)
        self.L.so.oc_opt_get(self.h, self.WHICH[name], ptr(out))
        return out

    def set(self, name: str, values) -> None:
        a = self.L.arr(values)
        assert a.shape == (self.d,)
        self.L.so.oc_opt_set(self.h, self.WHICH[name], ptr(a))

    def scalars(self) -> dict:
        Ln = len(self.sizes)
        out = np.zeros(3 * Ln, dtype=np.float64)
        self.L.so.oc_opt_get_scalars(self.h, ptr(out))
        return {"c_avg": out[:Ln].copy(), "r_prev": out[Ln:2 * Ln].copy(),
                "scale_coeff": out[2 * Ln:].copy()}

    def set_scalars(self, c_avg, r_prev) -> None:
        a = np.concatenate([np.asarray(c_avg, np.float64), np.asarray(r_prev, np.float64)])
        self.L.so.oc_opt_set_scalars(self.h, ptr(a))

    @property
    def frozen(self) -> bool:
        return bool(self.L.so.oc_opt_frozen(self.h))
