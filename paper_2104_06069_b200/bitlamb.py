"""Python mirror of the reference's communicator/optimizer API over the C-ABI.

Same names, argument meaning and error behaviour as the reference C++ library
(/root/reference/proj/include/bitlamb/comm_sim.hpp and optimizers.hpp), so the
parity tests read like the reference's own doctest suites.  Every call goes
through include/bitlamb_b200.h into libbitlamb_b200.so (hand-written sm_100a
kernels).  There is no CPU fallback: importing this module on a machine
without the library fails, and creating a cluster without a GPU raises.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
import sys
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BL_LIB_PATH: an alternative build of the same library (A/B timing).
LIB_PATH = os.environ.get("BL_LIB_PATH") or os.path.join(_HERE, "libbitlamb_b200.so")

# ---------------------------------------------------------------------------
# Exceptions: errors.hpp:26-53 (bl_status codes 1..6) + CUDA/NCCL/unsupported.
# ---------------------------------------------------------------------------


class BitlambError(Exception):
    status = 0


class DimensionError(BitlambError, ValueError):  # std::invalid_argument
    status = 1


class StageOrderError(BitlambError):  # std::logic_error
    status = 2


class ConfigError(BitlambError, RuntimeError):  # std::runtime_error
    status = 3


class InvalidArgument(BitlambError, ValueError):  # std::invalid_argument
    status = 4


class NumericalError(BitlambError, RuntimeError):  # std::runtime_error
    status = 5


class LogicError(BitlambError):  # std::logic_error
    status = 6


class CudaError(BitlambError, RuntimeError):
    status = 7


class NcclError(BitlambError, RuntimeError):
    status = 8


class Unsupported(BitlambError, NotImplementedError):
    status = 9


_ERRORS = {cls.status: cls for cls in (DimensionError, StageOrderError, ConfigError, InvalidArgument,
                                       NumericalError, LogicError, CudaError, NcclError, Unsupported)}

VARIANTS = {"lamb": 0, "adam": 1, "onebit_lamb": 2, "lamb_basic_1bit": 3, "onebit_adam": 4}
COMPRESSORS = {"onebit": 0, "identity": 1}
MEM_HOST, MEM_DEVICE = 0, 1
STATE = {"x": 0, "m": 1, "v": 2, "v_frozen": 3, "m_prev": 4}


class _ClusterConfig(C.Structure):
    _fields_ = [("n_workers", C.c_int32), ("mode", C.c_int32), ("rank", C.c_int32),
                ("device", C.c_int32), ("dim", C.c_uint64), ("compressor", C.c_int32),
                ("baseline_bits_per_element", C.c_int32), ("verify_compensation", C.c_int32),
                ("endpoint_stats", C.c_int32), ("compensation_tolerance", C.c_double),
                ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p), ("transport", C.c_int32)]


class _Ledger(C.Structure):
    _fields_ = [("gather_bits", C.c_uint64), ("scatter_bits", C.c_uint64),
                ("lossless_bits", C.c_uint64), ("baseline_equivalent_bits", C.c_uint64),
                ("compressed_collectives", C.c_uint64), ("lossless_collectives", C.c_uint64)]


class _Stats(C.Structure):
    _fields_ = [("delta_l2", C.c_double), ("delta_linf", C.c_double), ("corrected_linf", C.c_double),
                ("max_delta_linf", C.c_double), ("max_corrected_linf", C.c_double)]


class _HParams(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("beta1", "beta2", "beta3", "eta", "c_min", "c_max", "r_min",
                                          "r_max", "r_threshold", "weight_decay", "division_floor")] + \
               [("total_steps", C.c_uint64), ("warmup_steps", C.c_uint64),
                ("scaled_error_feedback", C.c_int32)]


class _LayerSpec(C.Structure):
    _fields_ = [("name", C.c_char_p), ("size", C.c_uint64)]


class _Trace(C.Structure):
    _fields_ = [("c", C.c_void_p), ("r", C.c_void_p), ("v_norm", C.c_void_p),
                ("v_ratio_preclip", C.c_void_p), ("compressed", C.c_int32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (or "
                          f"python paper_2104_06069_b200/build.py); there is no CPU fallback")
    so = C.CDLL(LIB_PATH)
    P, u64, i32 = C.c_void_p, C.c_uint64, C.c_int32
    so.bl_last_error.restype = C.c_char_p
    so.bl_abi_version.restype = i32
    so.bl_nccl_get_unique_id.argtypes = [P]
    so.bl_cluster_create.argtypes = [C.POINTER(_ClusterConfig), C.POINTER(P)]
    so.bl_cluster_destroy.argtypes = [P]
    so.bl_cluster_dims.argtypes = [P, C.POINTER(u64), C.POINTER(u64)]
    so.bl_cluster_transport.argtypes = [P]
    so.bl_cluster_transport.restype = i32
    so.bl_cluster_stream.argtypes = [P]
    so.bl_cluster_stream.restype = P
    so.bl_cluster_get_config.argtypes = [P, C.POINTER(_ClusterConfig)]
    so.bl_cluster_step_count.argtypes = [P]
    so.bl_cluster_step_count.restype = u64
    so.bl_cluster_set_peer_timeout.argtypes = [P, C.c_double]
    so.bl_optimizer_create_named.argtypes = [i32, P, i32, C.POINTER(_HParams), P, C.POINTER(P)]
    so.bl_optimizer_layer_name.argtypes = [P, i32]
    so.bl_optimizer_layer_name.restype = C.c_char_p
    so.bl_optimizer_set_strict.argtypes = [P, i32]
    so.bl_compress_with_feedback.argtypes = [P, P, u64, i32, C.c_double, P, P, i32, i32]
    so.bl_compute_scales.argtypes = [P, P, i32, C.c_double, P, P, i32, i32]
    so.bl_apply_scaling.argtypes = [P, P, i32, P, i32, i32]
    so.bl_remove_scaling.argtypes = [P, P, i32, P, i32, i32]
    so.bl_cluster_compressed_allreduce.argtypes = [P, P, i32, u64, P, C.c_double, i32]
    so.bl_cluster_lossless_allreduce.argtypes = [P, P, i32, u64, P, i32]
    so.bl_cluster_worker_error.argtypes = [P, i32, P]
    so.bl_cluster_server_error.argtypes = [P, i32, P]
    so.bl_cluster_packet.argtypes = [P, i32, i32, P]
    so.bl_cluster_server_packet.argtypes = [P, i32, P]
    so.bl_cluster_ledger.argtypes = [P, C.POINTER(_Ledger)]
    so.bl_cluster_stats.argtypes = [P, P]
    so.bl_cluster_synchronize.argtypes = [P]
    so.bl_cluster_input_buffer.argtypes = [P, i32]
    so.bl_cluster_input_buffer.restype = P
    so.bl_cluster_kernel_launches.argtypes = [P]
    so.bl_cluster_kernel_launches.restype = u64
    so.bl_cluster_compensation_checks.argtypes = [P]
    so.bl_cluster_compensation_checks.restype = u64
    so.bl_cluster_set_profiling.argtypes = [P, i32]
    so.bl_cluster_profile.argtypes = [P, P, P, P, i32]
    so.bl_cluster_profile.restype = i32
    so.bl_volume_reduction.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]
    so.bl_hparams_default.argtypes = [C.POINTER(_HParams)]
    so.bl_optimizer_create.argtypes = [i32, P, i32, C.POINTER(_HParams), P, C.POINTER(P)]
    so.bl_optimizer_destroy.argtypes = [P]
    so.bl_optimizer_step.argtypes = [P, P, P, i32, u64, C.c_double, i32, C.POINTER(_Trace)]
    so.bl_optimizer_grad_buffer.argtypes = [P, i32]
    so.bl_optimizer_grad_buffer.restype = P
    so.bl_optimizer_get_state.argtypes = [P, i32, P]
    so.bl_optimizer_set_state.argtypes = [P, i32, P]
    so.bl_optimizer_get_scalars.argtypes = [P, P, P, P]
    so.bl_optimizer_set_scalars.argtypes = [P, P, P]
    so.bl_optimizer_frozen.argtypes = [P]
    so.bl_optimizer_frozen.restype = i32
    so.bl_optimizer_fused_dim.argtypes = [P]
    so.bl_optimizer_fused_dim.restype = u64
    so.bl_optimizer_layer_count.argtypes = [P]
    so.bl_optimizer_layer_count.restype = i32
    return so


_lib = _load()
lib = _lib


def _check(status: int) -> None:
    if status != 0:
        msg = _lib.bl_last_error().decode(errors="replace")
        raise _ERRORS.get(status, BitlambError)(msg)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.bl_nccl_get_unique_id(buf))
    return bytes(buf)


def volume_reduction(warmup_ratio: float, baseline_bits: float,
                     compressed_bits_per_element: float) -> float:
    """comm_sim.hpp:55-56."""
    out = C.c_double()
    _check(_lib.bl_volume_reduction(warmup_ratio, baseline_bits, compressed_bits_per_element,
                                    C.byref(out)))
    return out.value


def compress_with_feedback(v, delta, kind: str = "onebit", error_scale: float = 1.0, device: int = 0):
    """compression.hpp:106-118 on the device.  `delta` (float32 numpy) is
    updated in place; returns (serialize() bytes or None, decompressed)."""
    v = np.ascontiguousarray(v, dtype=np.float32)
    if not (isinstance(delta, np.ndarray) and delta.dtype == np.float32 and delta.flags.c_contiguous):
        raise InvalidArgument("compress_with_feedback: delta must be a contiguous float32 array")
    if v.shape != delta.shape:
        raise DimensionError(f"compress_with_feedback: size mismatch ({v.size} vs {delta.size})")
    n = v.size
    wire = np.zeros((n + 7) // 8 + 4, dtype=np.uint8)
    dec = np.zeros(max(n, 1), dtype=np.float32)
    _check(_lib.bl_compress_with_feedback(v.ctypes.data, delta.ctypes.data, n, COMPRESSORS[kind],
                                          error_scale, wire.ctypes.data, dec.ctypes.data, MEM_HOST, device))
    return (wire.tobytes() if kind == "onebit" else None), dec[:n]


def _sizes(sizes) -> np.ndarray:
    return np.ascontiguousarray([int(x) for x in sizes], dtype=np.uint64)


def compute_scales(fused_m, sizes, floor: float = 1e-12, device: int = 0):
    """fusion.hpp:92-93: -> (coeff[L], reference_scale)."""
    m = np.ascontiguousarray(fused_m, dtype=np.float32)
    sz = _sizes(sizes)
    coeff = np.zeros(max(len(sz), 1), dtype=np.float64)
    ref = C.c_double()
    _check(_lib.bl_compute_scales(m.ctypes.data, sz.ctypes.data, len(sz), floor, coeff.ctypes.data,
                                  C.byref(ref), MEM_HOST, device))
    return coeff[: len(sz)], ref.value


def apply_scaling(fused, sizes, coeff, device: int = 0) -> np.ndarray:
    """fusion.hpp:96-98: returns fused * coeff per layer."""
    x = np.array(fused, dtype=np.float32, copy=True)
    sz = _sizes(sizes)
    co = np.ascontiguousarray(coeff, dtype=np.float64)
    if co.size != sz.size:
        raise DimensionError("apply_scaling: size mismatch")
    _check(_lib.bl_apply_scaling(x.ctypes.data, sz.ctypes.data, len(sz), co.ctypes.data, MEM_HOST, device))
    return x


def remove_scaling(fused, sizes, coeff, device: int = 0) -> np.ndarray:
    """fusion.hpp:100-102: returns fused * (1/coeff) per layer."""
    x = np.array(fused, dtype=np.float32, copy=True)
    sz = _sizes(sizes)
    co = np.ascontiguousarray(coeff, dtype=np.float64)
    if co.size != sz.size:
        raise DimensionError("remove_scaling: size mismatch")
    _check(_lib.bl_remove_scaling(x.ctypes.data, sz.ctypes.data, len(sz), co.ctypes.data, MEM_HOST, device))
    return x


@dataclass
class HyperParams:
    """optimizers.hpp:45-64 (paper defaults)."""

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

    def _c(self) -> _HParams:
        h = _HParams()
        for f in ("beta1", "beta2", "beta3", "eta", "c_min", "c_max", "r_min", "r_max", "r_threshold",
                  "weight_decay", "division_floor", "total_steps", "warmup_steps"):
            setattr(h, f, getattr(self, f))
        h.scaled_error_feedback = int(self.scaled_error_feedback)
        return h


@dataclass
class VolumeLedger:
    """comm_sim.hpp:37-50."""

    gather_bits: int = 0
    scatter_bits: int = 0
    lossless_bits: int = 0
    baseline_equivalent_bits: int = 0
    compressed_collectives: int = 0
    lossless_collectives: int = 0

    def total_sent_bits(self) -> int:
        return self.gather_bits + self.scatter_bits + self.lossless_bits

    def reduction_factor(self) -> float:
        sent = self.total_sent_bits()
        return 1.0 if sent == 0 else self.baseline_equivalent_bits / sent


@dataclass
class EndpointStats:
    delta_l2: float
    delta_linf: float
    corrected_linf: float
    max_delta_linf: float
    max_corrected_linf: float


@dataclass
class StepTrace:
    """optimizers.hpp:81-87."""

    c: np.ndarray
    r: np.ndarray
    v_norm: np.ndarray
    v_ratio_preclip: np.ndarray
    compressed: bool = False


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _torch_cuda_live() -> bool:
    """True once this process has touched CUDA through torch (its current
    stream may then hold pending writes into buffers the library reads)."""
    t = sys.modules.get("torch")
    return bool(t is not None and t.cuda.is_initialized())


class _DeviceView:
    """__cuda_array_interface__ over a library-owned device buffer, so torch
    can alias it without a copy (torch.as_tensor)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _pointers(inputs, length: int):
    """-> (ctypes array of pointers, memory kind, keepalive list)."""
    if _is_torch_cuda(inputs):
        inputs = [inputs[i] for i in range(inputs.shape[0])] if inputs.dim() == 2 else [inputs]
    elif isinstance(inputs, np.ndarray):
        inputs = [inputs] if inputs.ndim == 1 else [inputs[i] for i in range(inputs.shape[0])]
    items = list(inputs)
    keep = []
    ptrs = (C.c_void_p * max(1, len(items)))()
    dev = any(_is_torch_cuda(t) for t in items)
    for i, t in enumerate(items):
        if _is_torch_cuda(t):
            import torch

            if t.dtype != torch.float32 or not t.is_contiguous():
                t = t.to(torch.float32).contiguous()
            keep.append(t)
            ptrs[i] = t.data_ptr()
        else:
            a = np.ascontiguousarray(np.asarray(t), dtype=np.float32)
            keep.append(a)
            ptrs[i] = a.ctypes.data
    lens = {int(t.shape[-1]) for t in keep}
    if len(lens) > 1:  # comm_sim.cpp:124-126 checks every input's length
        bad = next(int(t.shape[-1]) for t in keep if int(t.shape[-1]) != length)
        raise DimensionError(f"input length: size mismatch ({bad} vs {length})")
    return ptrs, len(items), (MEM_DEVICE if dev else MEM_HOST), keep, (
        int(keep[0].shape[-1]) if keep else length)


class SimCluster:
    """bitlamb::SimCluster (comm_sim.hpp:72-148) on B200.

    mode="sim": n_workers ranks simulated in one GPU's HBM (the reference's
    in-process cluster).  mode="nccl": this process is `rank` of n_workers
    (one process per GPU); inputs/outputs are the local rank's."""

    def __init__(self, n_workers: int, dim: int, compressor: str = "onebit",
                 baseline_bits_per_element: int = 16, *, mode: str = "sim", rank: int = 0,
                 device: int = 0, nccl_unique_id: bytes | None = None, stream=None,
                 endpoint_stats: bool = False, verify_compensation: bool = False,
                 compensation_tolerance: float = 1e-12, transport: str = "auto"):
        cfg = _ClusterConfig()
        cfg.n_workers = n_workers
        cfg.mode = 0 if mode == "sim" else 1
        cfg.rank = rank
        cfg.device = device
        cfg.dim = dim
        cfg.compressor = COMPRESSORS[compressor]
        cfg.baseline_bits_per_element = baseline_bits_per_element
        cfg.verify_compensation = int(verify_compensation)
        cfg.endpoint_stats = int(endpoint_stats)
        cfg.compensation_tolerance = compensation_tolerance
        self._uid = None
        if nccl_unique_id is not None:
            self._uid = (C.c_uint8 * 128).from_buffer_copy(nccl_unique_id)
            cfg.nccl_unique_id = C.addressof(self._uid)
        cfg.stream = stream
        cfg.transport = {"auto": 0, "nccl": 1, "p2p": 2}[transport]
        h = C.c_void_p()
        _check(_lib.bl_cluster_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self.mode, self.rank, self.device = mode, rank, device
        self._n, self._dim = n_workers, dim
        p, c = C.c_uint64(), C.c_uint64()
        _check(_lib.bl_cluster_dims(self._h, C.byref(p), C.byref(c)))
        self.padded, self.chunk_len = p.value, c.value
        self._stream_ptr = int(_lib.bl_cluster_stream(self._h) or 0)
        self._ext = None

    @contextlib.contextmanager
    def torch_ordered(self, tensors=()):
        """Order the library's stream after torch's current stream on entry
        (inputs written by torch kernels) and torch's after the library's on
        exit (outputs read by torch kernels); torch temporaries handed to the
        library are recorded on its stream so the caching allocator does not
        reuse them while an asynchronous copy may still read them."""
        if not tensors and not _torch_cuda_live():
            yield
            return
        import torch

        dev = torch.device("cuda", self.device)
        if self._ext is None:
            self._ext = torch.cuda.ExternalStream(self._stream_ptr, device=dev)
        cur = torch.cuda.current_stream(dev)
        same = cur.cuda_stream == self._stream_ptr
        if not same:
            self._ext.wait_stream(cur)
        try:
            yield
        finally:
            if not same:
                cur.wait_stream(self._ext)
                for t in tensors:
                    if _is_torch_cuda(t):
                        t.record_stream(self._ext)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.bl_cluster_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def handle(self):
        return self._h

    @property
    def transport(self) -> str:
        """'sim', 'nccl' or 'p2p' (fused NVLink peer stores)."""
        if self.mode == "sim":
            return "sim"
        return {1: "nccl", 2: "p2p"}.get(int(_lib.bl_cluster_transport(self._h)), "nccl")

    def n_workers(self) -> int:
        return self._n

    def config(self) -> dict:
        """comm_sim.hpp:105."""
        c = _ClusterConfig()
        _check(_lib.bl_cluster_get_config(self._h, C.byref(c)))
        return {"n_workers": c.n_workers, "dim": c.dim,
                "compressor": {v: k for k, v in COMPRESSORS.items()}[c.compressor],
                "baseline_bits_per_element": c.baseline_bits_per_element,
                "verify_compensation": bool(c.verify_compensation),
                "compensation_tolerance": c.compensation_tolerance,
                "endpoint_stats": bool(c.endpoint_stats)}

    def step_count(self) -> int:
        """comm_sim.hpp:108 (compressed + lossless collectives)."""
        return int(_lib.bl_cluster_step_count(self._h))

    def set_peer_timeout(self, ms: float) -> None:
        _check(_lib.bl_cluster_set_peer_timeout(self._h, float(ms)))

    def dim(self) -> int:
        return self._dim

    def local_workers(self) -> int:
        return self._n if self.mode == "sim" else 1

    def input_buffer(self, worker: int) -> int:
        """Device pointer of worker's dim-float input buffer (zero-copy)."""
        return int(_lib.bl_cluster_input_buffer(self._h, worker))

    def compressed_allreduce(self, inputs, error_scale: float = 1.0, out=None):
        """comm_sim.hpp:98-99.  Returns the dim-long result (numpy for host
        inputs; writes `out` (a torch CUDA tensor) for device inputs)."""
        ptrs, n_in, mem, keep, length = _pointers(inputs, self._dim)
        if mem == MEM_DEVICE:
            import torch

            if out is None:
                out = torch.empty(self._dim, dtype=torch.float32, device=f"cuda:{self.device}")
            with self.torch_ordered(keep + [out]):
                _check(_lib.bl_cluster_compressed_allreduce(self._h, ptrs, n_in, length, out.data_ptr(),
                                                            error_scale, mem))
            return out
        res = np.zeros(max(self._dim, 1), dtype=np.float32)
        _check(_lib.bl_cluster_compressed_allreduce(self._h, ptrs, n_in, length, res.ctypes.data,
                                                    error_scale, mem))
        return res[: self._dim]

    def compressed_allreduce_resident(self, out, error_scale: float = 1.0):
        """compressed_allreduce on the streams already in the cluster's input
        buffers (zero-copy); `out` is a torch CUDA tensor of dim floats."""
        nw = self.local_workers()
        ptrs = (C.c_void_p * nw)(*[self.input_buffer(i) for i in range(nw)])
        with self.torch_ordered([out]):
            _check(_lib.bl_cluster_compressed_allreduce(self._h, ptrs, nw, self._dim, out.data_ptr(),
                                                        error_scale, MEM_DEVICE))
        return out

    def input_tensor(self, worker: int):
        """torch view (no copy) of worker's dim-float input buffer."""
        import torch

        return torch.as_tensor(_DeviceView(self.input_buffer(worker), self._dim),
                               device=f"cuda:{self.device}")

    def lossless_allreduce(self, inputs):
        """comm_sim.hpp:102."""
        ptrs, n_in, mem, keep, length = _pointers(inputs, self._dim)
        if mem == MEM_DEVICE:
            import torch

            out = torch.empty(self._dim, dtype=torch.float32, device=f"cuda:{self.device}")
            with self.torch_ordered(keep + [out]):
                _check(_lib.bl_cluster_lossless_allreduce(self._h, ptrs, n_in, length, out.data_ptr(),
                                                          mem))
            return out
        res = np.zeros(self._dim, dtype=np.float32)
        _check(_lib.bl_cluster_lossless_allreduce(self._h, ptrs, n_in, length, res.ctypes.data, mem))
        return res

    def worker_error(self, i: int) -> np.ndarray:
        out = np.zeros(self.padded, dtype=np.float32)
        _check(_lib.bl_cluster_worker_error(self._h, i, out.ctypes.data))
        return out

    def server_error(self, j: int) -> np.ndarray:
        out = np.zeros(self.chunk_len, dtype=np.float32)
        _check(_lib.bl_cluster_server_error(self._h, j, out.ctypes.data))
        return out

    def packet(self, worker: int, server: int) -> bytes:
        """CompressedBlock::serialize() bytes of worker's message to server."""
        out = np.zeros((self.chunk_len + 7) // 8 + 4, dtype=np.uint8)
        _check(_lib.bl_cluster_packet(self._h, worker, server, out.ctypes.data))
        return out.tobytes()

    def server_packet(self, server: int) -> bytes:
        out = np.zeros((self.chunk_len + 7) // 8 + 4, dtype=np.uint8)
        _check(_lib.bl_cluster_server_packet(self._h, server, out.ctypes.data))
        return out.tobytes()

    def ledger(self) -> VolumeLedger:
        led = _Ledger()
        _check(_lib.bl_cluster_ledger(self._h, C.byref(led)))
        return VolumeLedger(*[getattr(led, f) for f, _ in _Ledger._fields_])

    def _stats(self) -> list[EndpointStats]:
        arr = (_Stats * (2 * self._n))()
        _check(_lib.bl_cluster_stats(self._h, arr))
        return [EndpointStats(s.delta_l2, s.delta_linf, s.corrected_linf, s.max_delta_linf,
                              s.max_corrected_linf) for s in arr]

    def worker_stats(self) -> list[EndpointStats]:
        return self._stats()[: self._n]

    def server_stats(self) -> list[EndpointStats]:
        return self._stats()[self._n:]

    def delta_linf(self) -> float:
        return max(s.delta_linf for s in self._stats())

    def delta_l2_max(self) -> float:
        return max(s.delta_l2 for s in self._stats())

    def run_max_delta_linf(self) -> float:
        return max(s.max_delta_linf for s in self._stats())

    def run_max_corrected_linf(self) -> float:
        return max(s.max_corrected_linf for s in self._stats())

    def synchronize(self) -> None:
        _check(_lib.bl_cluster_synchronize(self._h))

    def compensation_checks(self) -> int:
        return int(_lib.bl_cluster_compensation_checks(self._h))

    def kernel_launches(self) -> int:
        return int(_lib.bl_cluster_kernel_launches(self._h))

    def set_profiling(self, on: bool) -> None:
        _check(_lib.bl_cluster_set_profiling(self._h, int(on)))

    def profile(self) -> dict:
        cap = 32
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        cnt = (C.c_uint64 * cap)()
        k = _lib.bl_cluster_profile(self._h, names, ms, cnt, cap)
        return {names[i].decode(): (ms[i], int(cnt[i])) for i in range(k)}


class Optimizer:
    """bitlamb::Optimizer (optimizers.hpp:93-145) on B200; state stays in HBM."""

    def __init__(self, variant: str, layout, hp: HyperParams, cluster: SimCluster, strict: bool = False):
        self.sizes = [int(s[1]) if isinstance(s, (tuple, list)) else int(s) for s in layout]
        self.names = [s[0] if isinstance(s, (tuple, list)) else f"layer{i}"
                      for i, s in enumerate(layout)]
        self.variant = variant
        self.hp = hp
        self.cluster = cluster
        self._names_b = [n.encode() for n in self.names]
        specs = (_LayerSpec * max(1, len(self.sizes)))()
        for i, (nm, sz) in enumerate(zip(self._names_b, self.sizes)):
            specs[i].name = nm
            specs[i].size = sz
        h = C.c_void_p()
        hpc = hp._c()
        _check(_lib.bl_optimizer_create_named(VARIANTS[variant], specs, len(self.sizes),
                                              C.byref(hpc), cluster.handle, C.byref(h)))
        self._h = h
        if strict:
            self.set_strict(True)
        self.offsets = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.bl_optimizer_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def fused_dim(self) -> int:
        return int(_lib.bl_optimizer_fused_dim(self._h))

    def set_strict(self, on: bool) -> None:
        """check_gradients (optimizers.cpp:99-117) before any state changes."""
        _check(_lib.bl_optimizer_set_strict(self._h, int(bool(on))))

    def layer_name(self, l: int) -> str:
        r = _lib.bl_optimizer_layer_name(self._h, l)
        if r is None:
            raise InvalidArgument("layer index out of range")
        return r.decode()

    def frozen(self) -> bool:
        return bool(_lib.bl_optimizer_frozen(self._h))

    def grad_buffer(self, worker: int) -> int:
        return int(_lib.bl_optimizer_grad_buffer(self._h, worker))

    def grad_tensor(self, worker: int):
        """torch view (no copy) of worker's device gradient buffer: write the
        gradient into it, then step_resident()."""
        import torch

        return torch.as_tensor(_DeviceView(self.grad_buffer(worker), self.fused_dim()),
                               device=f"cuda:{self.cluster.device}")

    def _fuse(self, local_grads):
        """[worker][layer] arrays, [worker] fused arrays, or a 2-D array."""
        if isinstance(local_grads, np.ndarray) or _is_torch_cuda(local_grads):
            return local_grads
        out = []
        for w in local_grads:
            if isinstance(w, (list, tuple)):
                out.append(np.concatenate([np.asarray(a, dtype=np.float32).ravel() for a in w]))
            else:
                out.append(w)
        return out

    def step(self, local_grads, t: int, lr: float, cluster: SimCluster | None = None,
             trace: bool = True) -> StepTrace | None:
        """optimizers.hpp:106-107.  trace=False runs fully asynchronously."""
        cluster = cluster or self.cluster
        ptrs, n_in, mem, keep, length = _pointers(self._fuse(local_grads), self.fused_dim())
        if length != self.fused_dim() and n_in > 0:
            raise DimensionError(f"step: gradient length: size mismatch ({length} vs {self.fused_dim()})")
        L = len(self.sizes)
        if not trace:
            with cluster.torch_ordered(keep if mem == MEM_DEVICE else ()):
                _check(_lib.bl_optimizer_step(self._h, cluster.handle, ptrs, n_in, t, lr, mem, None))
            return None
        arrs = [np.zeros(L, dtype=np.float64) for _ in range(4)]
        tr = _Trace(*[a.ctypes.data for a in arrs], 0)
        with cluster.torch_ordered(keep if mem == MEM_DEVICE else ()):
            _check(_lib.bl_optimizer_step(self._h, cluster.handle, ptrs, n_in, t, lr, mem, C.byref(tr)))
        return StepTrace(arrs[0], arrs[1], arrs[2], arrs[3], bool(tr.compressed))

    def step_resident(self, t: int, lr: float, trace: bool = False) -> StepTrace | None:
        """Step on the gradients already in the device grad buffers (zero-copy)."""
        nw = self.cluster.local_workers()
        ptrs = (C.c_void_p * nw)(*[self.grad_buffer(i) for i in range(nw)])
        return self._step_ptrs(ptrs, nw, t, lr, MEM_DEVICE, trace)

    def step_host_pointers(self, ptrs: Sequence[int], t: int, lr: float,
                           trace: bool = True) -> StepTrace | None:
        """Step on host (pinned) gradient buffers given as raw pointers."""
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        return self._step_ptrs(arr, len(ptrs), t, lr, MEM_HOST, trace)

    def _step_ptrs(self, ptrs, n, t, lr, mem, trace):
        L = len(self.sizes)
        if not trace:
            with self.cluster.torch_ordered():
                _check(_lib.bl_optimizer_step(self._h, self.cluster.handle, ptrs, n, t, lr, mem, None))
            return None
        arrs = [np.zeros(L, dtype=np.float64) for _ in range(4)]
        tr = _Trace(*[a.ctypes.data for a in arrs], 0)
        with self.cluster.torch_ordered():
            _check(_lib.bl_optimizer_step(self._h, self.cluster.handle, ptrs, n, t, lr, mem, C.byref(tr)))
        return StepTrace(arrs[0], arrs[1], arrs[2], arrs[3], bool(tr.compressed))

    def get(self, name: str) -> np.ndarray:
        out = np.zeros(self.fused_dim(), dtype=np.float32)
        _check(_lib.bl_optimizer_get_state(self._h, STATE[name], out.ctypes.data))
        return out

    def set(self, name: str, values) -> None:
        a = np.ascontiguousarray(values, dtype=np.float32)
        if a.shape != (self.fused_dim(),):
            raise DimensionError("set: size mismatch")
        _check(_lib.bl_optimizer_set_state(self._h, STATE[name], a.ctypes.data))

    def layer(self, name: str, l: int) -> np.ndarray:
        return self.get(name)[self.offsets[l]:self.offsets[l + 1]]

    def scalars(self) -> dict:
        L = len(self.sizes)
        c_avg, r_prev, coeff = (np.zeros(L) for _ in range(3))
        _check(_lib.bl_optimizer_get_scalars(self._h, c_avg.ctypes.data, r_prev.ctypes.data,
                                             coeff.ctypes.data))
        return {"c_avg": c_avg, "r_prev": r_prev, "scale_coeff": coeff}

    def set_scalars(self, c_avg=None, r_prev=None) -> None:
        a = None if c_avg is None else np.ascontiguousarray(c_avg, dtype=np.float64)
        b = None if r_prev is None else np.ascontiguousarray(r_prev, dtype=np.float64)
        _check(_lib.bl_optimizer_set_scalars(self._h, None if a is None else a.ctypes.data,
                                             None if b is None else b.ctypes.data))

    def momentum_scales(self) -> np.ndarray:
        return self.scalars()["scale_coeff"]
