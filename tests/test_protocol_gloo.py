"""world_size-2 CPU (gloo) tests of the sharded path's host logic.

The NCCL-mode cluster shards the collective exactly as the reference's
role assignment does (comm_sim.hpp:61-69: worker i serves chunk i): every
rank compresses its own stream's n chunks, sends chunk j's packet to rank j
(alltoall), reduces the n packets of its own chunk, and allgathers the server
packets.  Here two gloo processes run that protocol with the f32 oracle's
per-rank phases and the package's rendezvous helpers; the result must equal
the in-process n-worker simulation bit-for-bit, step after step.
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank: int, world: int, port: int, d: int, steps: int, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C

        from oracle import oracle as O
        from paper_2104_06069_b200 import distributed as D

        L = O.lib("f32")
        padded = -(-d // world) * world
        c = padded // world
        ipk = (c + 7) // 8 + 4  # f32 in-memory packet == serialize() layout
        werr = np.zeros(padded, np.float32)
        serr = np.zeros(c, np.float32)
        b0, b1 = D.chunk_bounds(d, world, rank)
        assert b1 - b0 == c and D.packet_bytes(c) == ipk
        # the rendezvous helper moves a (fake) 128-byte NCCL id unchanged
        uid = D.new_unique_id(generate=lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        results = []
        for step in range(steps):
            streams = np.random.default_rng(1000 + step).standard_normal((world, d)).astype(np.float32)
            mine = np.ascontiguousarray(streams[rank])
            pk = np.zeros(world * ipk, np.uint8)
            L.check(L.so.oc_worker_compress(mine.ctypes.data, d, world, werr.ctypes.data, 1.0,
                                            pk.ctypes.data))
            recv = torch.empty(world * ipk, dtype=torch.uint8)
            dist.all_to_all_single(recv, torch.from_numpy(pk))  # packet (i -> j) to rank j
            sp = np.zeros(ipk, np.uint8)
            rbuf = recv.numpy().copy()
            L.check(L.so.oc_server_reduce(rbuf.ctypes.data, c, world, serr.ctypes.data, 1.0,
                                          sp.ctypes.data))
            gathered = [torch.empty(ipk, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(sp))
            out = np.zeros(padded, np.float32)
            for j, g in enumerate(gathered):
                gb = g.numpy().copy()
                L.so.oc_decompress(gb.ctypes.data, c, out[j * c:].ctypes.data)
            results.append(out[:d].copy())
        t = D.max_over_ranks(float(rank + 1))
        q.put((rank, results, werr, serr, t))
    except Exception as exc:  # surface the failure to the parent
        q.put((rank, repr(exc), None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d", [5, 37, 9001])
def test_two_rank_protocol_matches_simulation(d):
    world, steps = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        r, res, werr, serr, t = q.get(timeout=120)
        assert not isinstance(res, str), res
        got[r] = (res, werr, serr, t)
    for p in procs:
        p.join(timeout=60)
    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    sim = O.Cluster("f32", world, d)
    for step in range(steps):
        streams = np.random.default_rng(1000 + step).standard_normal((world, d)).astype(np.float32)
        ref = sim.compressed_allreduce(streams)
        for r in range(world):
            np.testing.assert_array_equal(got[r][0][step], ref)
    for r in range(world):
        np.testing.assert_array_equal(got[r][1], sim.worker_error(r))
        np.testing.assert_array_equal(got[r][2], sim.server_error(r))
        assert got[r][3] == float(world)  # max over ranks
