"""Compressed-allreduce message-size sweep vs fp32 NCCL allreduce (BASELINE
config 5).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench_sweep.py [--sizes-mb 1,4,...]

For each flat fp32 buffer of M MB (d = M * 2^18 elements, one layer), each
rank times SimCluster::compressed_allreduce (comm_sim.hpp:98-99) on its own
device-resident stream: K1 -> fused NVLink exchange (or NCCL) -> K3 ->
exchange -> decompress into the fp32 result.  It then times
torch.distributed.all_reduce (NCCL, fp32 sum) on the same buffer.  Times use
CUDA events and take the max over ranks.  Rank 0 prints one JSON line per
size with algbw = 4d / t for both.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2104_06069_b200 import bitlamb as bl  # noqa: E402
from paper_2104_06069_b200 import distributed as D  # noqa: E402


def timed(fn, stream, iters: int) -> float:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    a.record(stream)
    for _ in range(iters):
        fn()
    b.record(stream)
    b.synchronize()
    return D.max_over_ranks(a.elapsed_time(b) / iters)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mb", default="1,4,16,64,256,1024,4096")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"])
    args = ap.parse_args()
    rank, world, local = D.env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # A real stream: the default stream's handle is NULL, which the library
    # would replace by its own stream, escaping the events below.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    for mb in [int(x) for x in args.sizes_mb.split(",")]:
        d = mb * (1 << 18)
        x = torch.randn(d, device="cuda", dtype=torch.float32)
        out = torch.empty(d, device="cuda", dtype=torch.float32)
        cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local,
                           nccl_unique_id=D.new_unique_id(), stream=stream.cuda_stream,
                           transport=args.transport)
        # stage the input once into the cluster's own buffer; the timed calls
        # are zero-copy (the stream is read where it lives, like NCCL in place)
        cl.compressed_allreduce(x, out=out)

        def comp():
            cl.compressed_allreduce_resident(out)

        for _ in range(3):
            comp()
        t_c = timed(comp, stream, args.iters)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        for _ in range(args.iters):
            comp()
        host_us = (time.perf_counter() - h0) * 1e6 / args.iters  # enqueue cost per call
        torch.cuda.synchronize()
        cl.set_profiling(True)
        for _ in range(3):
            comp()
        prof = {k: round(v[0] / max(v[1], 1), 4) for k, v in cl.profile().items()}
        cl.set_profiling(False)
        y = x.clone()

        def nccl():
            dist.all_reduce(y)

        for _ in range(3):
            nccl()
        t_n = timed(nccl, stream, args.iters)
        if rank == 0:
            print(json.dumps({
                "metric": "compressed_allreduce vs fp32 ncclAllReduce", "size_mb": mb, "elements": d,
                "n_gpus": world, "transport": cl.transport,
                "compressed_ms": t_c, "compressed_algbw_gbs": 4 * d / (t_c * 1e-3) / 1e9,
                "nccl_fp32_ms": t_n, "nccl_fp32_algbw_gbs": 4 * d / (t_n * 1e-3) / 1e9,
                "speedup": t_n / t_c, "kernels_ms": prof, "host_enqueue_us": host_us,
                "note": "compressed: zero-copy input, includes the fp32 decompress into the output",
            }), flush=True)
        cl.close()
        del x, y, out
        torch.cuda.empty_cache()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
