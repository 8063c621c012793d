"""Benchmark: compression-stage 1-bit LAMB step on a BERT-Large-shaped buffer.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 runs one rank in-process; N>1 is launched by torchrun, one process per
GPU, ranks exchanging packets over NCCL (weak scaling: every rank holds the
full 336M-parameter replica and its own gradient, as in data parallelism).

One "step" = Optimizer::step in the compression stage (optimizers.cpp:231-332):
K1 worker compress -> alltoall -> K3 server reduce -> allgather -> K5/K6
update.  `value` times K steps on device-resident gradients with CUDA events
on the library's stream (max over ranks); `e2e` times the same step through
the C-ABI with the gradient in pinned HOST memory (H2D copy + trace D2H inside
the timed region).  The reference arm runs the reference library itself
(oracle/_ref: the unmodified reference sources, fp64, OpenMP over every host
core) on the SAME full layout and worker count; it times as many of the
requested steps as fit a bounded budget and reports the steps it timed.
Both arms print the identical `config` object.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2104_06069_b200 import layouts  # noqa: E402

METRIC = "1-bit LAMB compression-stage step time, BERT-Large params (336,226,108)"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def hbm_peak() -> tuple[float, str]:
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def grad_sigma(sizes, seed=1):
    """Per-tensor gradient scale 10^(-4+2u) (SURVEY §8(d) synthetic inputs)."""
    u = np.random.default_rng(seed).random(len(sizes))
    return 10.0 ** (-4 + 2 * u)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and throttle reasons every ~5 ms through NVML while the
    timed region runs (nvidia-smi's 100 ms floor is too coarse for it)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None

    def _run(self):
        import pynvml as N

        while not self._stop.is_set():
            try:
                self.samples.append((float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)),
                                     int(N.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        import threading

        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as N

            N.nvmlInit()
            self.h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            time.sleep(0.02)
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self) -> dict:
        sm = [c for c, _ in self.samples]
        mask = 0
        for _, r in self.samples:
            mask |= r
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                "samples": len(sm), "reasons": sorted(k for k, b in self.REASONS.items() if mask & b)}


# ---------------------------------------------------------------------------
# algorithmic bytes per launch
# ---------------------------------------------------------------------------
def algorithmic_bytes(d: int, n: int, nw: int, share: float = 1.0) -> dict:
    """HBM bytes per step of each kernel (all its sub-launches); `share` is the
    fraction of the tiles a rank updates in the warmup stage (1/n when the
    multi-process warmup is owner-sharded)."""
    P = -(-d // n) * n
    c = P // n
    ns = nw
    return {
        # warmup stage: W1 g, m r/w, v r/w, x (24d); W2 m, v, x r/w (16d)
        "w1_warmup_a": 24 * d * share,
        "w2_warmup_b": 16 * d * share,
        # g (4d) + werr r/w (8P) + prev worker packet, prev result packet, new packet (3P/8)
        "k1_worker_compress": nw * (4 * d + 8 * P + 3 * P / 8),
        # serr r/w (8c) + n worker packets + prev server packet + new packet
        "k3_server_reduce": ns * (8 * c + (n + 2) * c / 8),
        # v r/w, vf (12d) + current and previous result bits (d/4)
        "k5_update_a": 12 * d + d / 4,
        # x r/w, vf (12d) + current result bits (d/8)
        "k6_update_b": 12 * d + d / 8,
    }


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the reference library on the host cores
# ---------------------------------------------------------------------------
def cpu_cores() -> int:
    """Host threads given to the reference: BL_REF_THREADS, else every core
    (torchrun exports OMP_NUM_THREADS=1, which must not throttle the baseline)."""
    return int(os.environ.get("BL_REF_THREADS", os.cpu_count() or 1))


def reference_run(layout, n: int, steps: int, warmup: int, budget_s: float) -> dict:
    """The reference's own compression-stage Optimizer::step (optimizers.cpp:
    334-364; oracle/_ref = the unmodified reference sources, fp64, OpenMP over
    the host cores) on the FULL layout with n simulated workers.

    Warm start: one warmup LAMB step that freezes (T_w = 1), then up to
    `warmup` untimed compression steps, then up to `steps` timed ones.  Each
    step is timed in C++ around the stock call alone (gradients already in the
    reference's [worker][layer] form, as our arm's are resident in HBM).  The
    timed steps stop early once their total would pass `budget_s`; the line
    reports the steps actually timed."""
    from oracle import oracle as O

    sizes = layouts.sizes(layout)
    d = sum(sizes)
    cores = O.set_reference_threads(cpu_cores())
    rng = np.random.default_rng(1)
    hp = O.HyperParams(total_steps=2 + warmup + steps, warmup_steps=1)
    cl = O.Cluster("ref", n, d)
    opt = O.Optimizer("ref", "onebit_lamb", sizes, hp)
    opt.set("x", rng.standard_normal(d, dtype=np.float32) * np.float32(0.02))
    sig = np.repeat(grad_sigma(sizes), sizes).astype(np.float32)
    g = np.empty((n, d), dtype=np.float64)
    for i in range(n):
        g[i] = rng.standard_normal(d, dtype=np.float32) * sig
    del sig
    opt.load_grads(g)
    del g
    lr = 1e-3
    opt.step_loaded(0, lr, cl)  # warmup LAMB + finalize_warmup (freeze)
    t, warm_done = 1, 0
    for _ in range(max(0, warmup)):
        opt.step_loaded(t, lr, cl)
        t, warm_done = t + 1, warm_done + 1
    times = []
    while len(times) < max(1, steps):
        sec, comp = opt.step_loaded(t, lr, cl)
        assert comp, "reference step did not run the compression stage"
        times.append(sec)
        t += 1
        if sum(times) + sum(times) / len(times) > budget_s:
            break
    ms = 1e3 * sum(times) / len(times)
    sample = (f"reference Optimizer::step, compression stage, full layout ({d:,} params, "
              f"{len(sizes)} tensors), {n} simulated worker(s); {len(times)} timed step(s) "
              f"(mean; requested {steps}) after 1 warmup LAMB step + freeze and {warm_done} untimed "
              f"compression step(s); {cores} OpenMP threads")
    return {"value": ms, "unit": "ms", "cores": cores, "kind": "reference", "sample": sample,
            "steps_timed": len(times), "warmup_done": 1 + warm_done,
            "step_ms": [1e3 * x for x in times]}


def workload_config(args, d: int, n_layers: int, world: int) -> dict:
    """The `config` object both arms print (identical by construction)."""
    return {"workload": f"{args.workload} 1-bit LAMB {args.stage}-stage step",
            "params": d, "layers": n_layers, "world": world, "parallelism": f"dp{world}",
            "l2": (f"inputs larger than L2 ({4 * d / 1e9:.2f} GB per state buffer vs 126 MB L2)"
                   if 4 * d > 126e6 else
                   f"state buffers ({4 * d / 1e6:.0f} MB each) fit in the 126 MB L2; no flush")}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bert-large", choices=["bert-large", "bert-base", "config1"])
    ap.add_argument("--sim-workers", type=int, default=0,
                    help="simulate this many ranks on one GPU instead of one rank per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="reference arm: stop timing steps once their total passes this many seconds")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"],
                    help="NCCL-mode packet exchange: fused NVLink peer stores or NCCL")
    ap.add_argument("--stage", default="compression", choices=["compression", "warmup"],
                    help="time compression-stage steps (headline) or warmup LAMB steps")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "W >= 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    layout = {"bert-large": layouts.bert_large, "bert-base": layouts.bert_base,
              "config1": lambda: [(f"l{i}", s) for i, s in enumerate(layouts.CONFIG1)]}[args.workload]()
    sizes = layouts.sizes(layout)
    d = sum(sizes)
    n = args.sim_workers if args.sim_workers else max(world, args.gpus if world == 1 else world)
    if world == 1 and not args.sim_workers:
        n = 1

    if args.impl == "reference":
        if rank != 0:
            return
        if args.stage != "compression":
            print(json.dumps({"impl": "reference", "unavailable": "reference arm times the compression stage"}))
            return
        ref = reference_run(layout, n, args.steps, min(args.warmup, 1), budget_s=args.ref_budget)
        line = {"impl": "reference",
                "metric": METRIC if args.workload == "bert-large" else f"1-bit LAMB step time, {args.workload}",
                "value": ref["value"], "unit": "ms",
                "n_gpus": args.gpus if world == 1 else world,
                # the steps actually timed / run untimed (requested: steps_requested, warmup_requested)
                "steps": ref["steps_timed"], "warmup": ref["warmup_done"],
                "steps_requested": args.steps, "warmup_requested": args.warmup,
                "ms_per_step": ref["value"], "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(args, d, len(sizes), n),
                "placement": {"mode": "reference CPU library, simulated workers", "cores": ref["cores"]},
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "step_ms": ref["step_ms"],
                "e2e": {"value": ref["value"], "unit": "ms", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2104_06069_b200 import bitlamb as bl

    stream = torch.cuda.Stream(device=local)
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(bl.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local,
                           nccl_unique_id=bytes(uid.cpu().numpy().tobytes()),
                           stream=stream.cuda_stream, transport=args.transport)
    else:
        cl = bl.SimCluster(n, d, device=local, stream=stream.cuda_stream)
    nw = cl.local_workers()
    total_steps = 2 + args.warmup + 2 * args.steps + 8
    hp = bl.HyperParams(total_steps=total_steps,
                        warmup_steps=2 if args.stage == "compression" else total_steps)
    opt = bl.Optimizer("onebit_lamb", layout, hp, cl)

    # synthetic state and gradients (x0 ~ N(0, 0.02^2); g ~ N(0, sigma_l^2))
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    x0 = (torch.randn(d, generator=gen, device="cuda") * 0.02).cpu().numpy()
    opt.set("x", x0)
    sig = torch.from_numpy(np.repeat(grad_sigma(sizes), sizes).astype(np.float32)).cuda()
    grads = torch.randn((nw, d), generator=gen, device="cuda") * sig
    del sig
    torch.cuda.synchronize()

    # warm start: 2 warmup LAMB steps (freeze at the end), then compression steps
    t = 0
    for _ in range(2):
        opt.step(grads, t, 1e-3)
        t += 1
    for _ in range(args.warmup):
        opt.step(grads, t, 1e-3, trace=False)  # copies grads into the resident buffer
        t += 1
    cl.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if not dist:
            return v
        tt = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # ---- timed region: device-resident gradients ----
    l0 = cl.kernel_launches()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        start.record(stream)
        for _ in range(args.steps):
            opt.step_resident(t, 1e-3)
            t += 1
        stop.record(stream)
        stop.synchronize()
    cl.synchronize()
    barrier()
    launches = (cl.kernel_launches() - l0) // args.steps
    ms = max_over_ranks(start.elapsed_time(stop) / args.steps)

    # ---- per-kernel breakdown (separate profiled pass, same steps) ----
    cl.set_profiling(True)
    for _ in range(args.steps):
        opt.step_resident(t, 1e-3)
        t += 1
    prof = cl.profile()
    cl.set_profiling(False)
    kern = {k: {"ms_per_launch": v[0] / max(v[1], 1), "launches": v[1]} for k, v in prof.items()}
    # Owner-sharded warmup (multi-process over NVLink): a rank updates 1/n of the tiles.
    sharded = (args.stage == "warmup" and world > 1 and cl.transport == "p2p"
               and os.environ.get("BL_WARMUP_SHARD", "1") != "0")
    ab = algorithmic_bytes(d, cl.n_workers(), nw, 1.0 / world if sharded else 1.0)
    peak, peak_kind = hbm_peak()

    def step_ms(k):  # a kernel's time per step, summed over its sub-launches
        return kern[k]["ms_per_launch"] * kern[k]["launches"] / args.steps

    dom = max((k for k in kern if k in ab), key=step_ms)
    achieved = ab[dom] / (step_ms(dom) * 1e-3) / 1e9
    traffic, traffic_src = None, None
    import glob

    caps = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    final = os.path.join(ROOT, "profiles", "round2_final_traffic.json")  # the end-of-round capture
    if os.path.exists(final):
        caps.append(final)
    if caps and args.workload == "bert-large" and cl.n_workers() == 1:
        with open(caps[-1]) as f:
            tj = json.load(f)
        if dom in tj:
            traffic = tj[dom]["dram_bytes"]
            traffic_src = os.path.relpath(caps[-1], ROOT)
    for k in kern:
        if k in ab:
            kern[k]["gbs"] = ab[k] / (step_ms(k) * 1e-3) / 1e9
    comm_ms = sum(kern.get(k, {}).get("ms_per_launch", 0) * kern.get(k, {}).get("launches", 0)
                  for k in ("k1_worker_compress", "finalize_scales", "nccl_alltoall", "k3_server_reduce",
                            "nccl_allgather")) / args.steps

    # ---- e2e: reference-facing C-ABI call with pinned host gradients ----
    e2e = None
    if not args.no_e2e:
        host = torch.empty((nw, d), dtype=torch.float32, pin_memory=True)
        host.copy_(grads)
        ptrs = [host[i].data_ptr() for i in range(nw)]
        opt.step_host_pointers(ptrs, t, 1e-3)  # warm
        t += 1
        barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            opt.step_host_pointers(ptrs, t, 1e-3)  # H2D + step + trace D2H (synchronous)
            t += 1
        e1.record(stream)
        e1.synchronize()
        wall = (time.perf_counter() - t0) * 1e3 / args.steps
        e2e_ms = max_over_ranks(max(e0.elapsed_time(e1) / args.steps, wall))
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 4 * d * nw,
               "d2h_bytes_per_step": 4 * len(sizes) * 8 + 32}

    del grads
    torch.cuda.empty_cache()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.stage == "compression":
        try:  # one timed reference step on the same full layout (bounded: ~1 min of CPU work)
            ref = reference_run(layout, cl.n_workers(), 1, 1, budget_s=0.0)
            cpu = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # reported, never silently replaced
            cpu = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {
            "metric": (METRIC if args.workload == "bert-large" else f"1-bit LAMB step time, {args.workload}")
            if args.stage == "compression" else f"warmup LAMB step time, {args.workload}",
            "value": ms, "unit": "ms", "n_gpus": args.gpus if world == 1 else world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, d, len(sizes), cl.n_workers()),
            "placement": {"mode": "nccl" if world > 1 else ("sim" if n > 1 else "single"),
                          "transport": cl.transport},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes": ab[dom]},
            "kernels": kern,
            "compressed_allreduce_ms": comm_ms,
            # warmup stage over NVLink: the all-reduce moves 2 (n-1)/n * 4d bytes per
            # direction per rank (reduce-scatter reads + allgather stores)
            "warmup_nvlink_gbs_per_direction": (2 * (world - 1) / world * 4 * d / (ms * 1e-3) / 1e9)
            if args.stage == "warmup" and world > 1 else None,
            "warmup_sharded": sharded,
            "compressed_allreduce_algbw_gbs": 4 * d / (comm_ms * 1e-3) / 1e9 if comm_ms else None,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
