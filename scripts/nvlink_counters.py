"""NVLink bytes per step from the hardware counters (NVML), under torchrun.

ncu cannot replay kernels that wait on another rank, so the fused NVLink
kernels (k_lossless_p2p, the LL small collective, K1/K3 peer stores) are
measured with the NVLink data-throughput counters instead
(NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES per link, summed):
read before and after K synchronized steps of one workload, on every rank.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/nvlink_counters.py

Rank 0 prints one JSON line per workload with TX/RX bytes per step per rank
(max over ranks) next to the algorithmic NVLink bytes of DESIGN.md §6.
"""
from __future__ import annotations

import json
import os
import sys
import time
from ctypes import byref

import numpy as np
import pynvml as N
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2104_06069_b200 import bitlamb as bl  # noqa: E402
from paper_2104_06069_b200 import distributed as D  # noqa: E402
from paper_2104_06069_b200 import layouts  # noqa: E402


def counters(h) -> tuple[int, int]:
    """(transmitted, received) bytes summed over the GPU's NVLinks.  The
    per-link byte counters (NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES, scope =
    link) are used where supported; else the data-throughput counters (KiB)."""
    ids = []
    for link in range(18):
        ids += [(N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, link), (N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, link)]
    vals = N.nvmlDeviceGetFieldValues(h, ids)
    tx = rx = 0
    good = 0
    for k, v in enumerate(vals):
        if v.nvmlReturn != 0:
            continue
        good += 1
        if k % 2 == 0:
            tx += int(v.value.ullVal)
        else:
            rx += int(v.value.ullVal)
    if good:
        return tx, rx
    vals = N.nvmlDeviceGetFieldValues(h, [N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                          N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
    out = []
    for v in vals:
        if v.nvmlReturn != 0:
            raise RuntimeError(f"no NVLink byte counter is readable (NVML {v.nvmlReturn})")
        out.append(int(v.value.ullVal) * 1024)
    return out[0], out[1]


class Gpm:
    """NVLink TX/RX through GPU performance monitoring (NVML GPM): the
    average NVLink bytes/s between two samples, times the interval."""

    def __init__(self, h):
        self.h = h
        self.a, self.b = N.nvmlGpmSampleAlloc(), N.nvmlGpmSampleAlloc()

    def start(self):
        self.t0 = time.perf_counter()
        N.nvmlGpmSampleGet(self.h, self.a)

    def stop(self) -> tuple[float, float]:
        N.nvmlGpmSampleGet(self.h, self.b)
        dt = time.perf_counter() - self.t0
        mg = N.c_nvmlGpmMetricsGet_t()
        mg.version = N.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1, mg.sample2 = self.a, self.b
        mg.metrics[0].metricId = N.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        mg.metrics[1].metricId = N.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        N.nvmlGpmMetricsGet(mg)
        for k in range(2):
            if mg.metrics[k].nvmlReturn != 0:
                raise RuntimeError(f"GPM NVLink metric unsupported (NVML {mg.metrics[k].nvmlReturn})")
        return mg.metrics[0].value * dt, mg.metrics[1].value * dt


def measure(h, fn, steps: int) -> tuple[float, float]:
    torch.cuda.synchronize()
    dist.barrier()
    try:
        tx0, rx0 = counters(h)
        gpm = None
    except RuntimeError:
        gpm = Gpm(h)
        gpm.start()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    if gpm is None:
        tx1, rx1 = counters(h)
        tx, rx = tx1 - tx0, rx1 - rx0
    else:
        tx, rx = gpm.stop()
    dist.barrier()
    return D.max_over_ranks(tx / steps), D.max_over_ranks(rx / steps)


def main():
    rank, world, local = D.env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    steps = 10
    rows = []

    # BERT-Large optimizer steps: warmup (lossless NVLink all-reduce) and compression stage
    layout = layouts.bert_large()
    sizes = layouts.sizes(layout)
    d = sum(sizes)
    cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=D.new_unique_id(),
                       stream=stream.cuda_stream)
    total = 4 + 2 * steps
    opt = bl.Optimizer("onebit_lamb", layout, bl.HyperParams(total_steps=total, warmup_steps=steps + 1), cl)
    g = torch.randn(d, device="cuda") * 1e-3
    opt.grad_tensor(0).copy_(g)
    del g
    t = [0]

    def step():
        opt.step_resident(t[0], 1e-3)
        t[0] += 1

    step()
    tx, rx = measure(h, step, steps)  # warmup steps (freeze comes after)
    c = -(-d // world)
    rows.append({"workload": "bert-large warmup step (k_lossless_p2p)", "tx_bytes": tx, "rx_bytes": rx,
                 "algorithmic_bytes_per_direction": 2 * (world - 1) * c * 4})
    step()  # the freezing step
    step()  # first compression step
    tx, rx = measure(h, step, steps)
    W = -(-c // 4096) * 4096 // 32
    rows.append({"workload": "bert-large compression step (K1/K3 peer stores)", "tx_bytes": tx, "rx_bytes": rx,
                 "algorithmic_bytes_per_direction": 2 * (world - 1) * (c + 7) // 8})
    opt.close()
    cl.close()

    # compressed_allreduce API: the LL small collective and the split kernels
    for mb in (1, 16, 256):
        dd = mb << 18
        x = torch.randn(dd, device="cuda")
        out = torch.empty_like(x)
        cl = bl.SimCluster(world, dd, mode="nccl", rank=rank, device=local, nccl_unique_id=D.new_unique_id(),
                           stream=stream.cuda_stream)
        cl.compressed_allreduce(x, out=out)
        tx, rx = measure(h, lambda: cl.compressed_allreduce_resident(out), steps)
        cc = -(-dd // world)
        rows.append({"workload": f"compressed_allreduce {mb} MB", "tx_bytes": tx, "rx_bytes": rx,
                     "algorithmic_bytes_per_direction": 2 * (world - 1) * (cc + 7) // 8,
                     "note": "LL small collective: each 4-byte word travels with its epoch (8 B)"
                     if (world * (-(-cc // 4096))) <= 2048 else "separate kernels"})
        cl.close()
    if rank == 0:
        for r in rows:
            r.update({"n_gpus": world, "steps": steps,
                      "tx_over_algorithmic": r["tx_bytes"] / max(r["algorithmic_bytes_per_direction"], 1)})
            print(json.dumps(r), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
