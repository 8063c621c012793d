"""Multi-GPU parity check (run under torchrun, one process per GPU).

Every rank runs the NCCL-mode cluster/optimizer on its own GPU with its own
gradient; rank 0 additionally runs the same n-worker job in SIM mode on its
GPU.  The real collective must reproduce the simulated one bit-for-bit:
worker packets, server packets, residuals, results, and the replicated
optimizer state after every step (warmup with the deterministic lossless
all-reduce, freeze, compression stage).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/multigpu_check.py
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2104_06069_b200 import bitlamb as bl  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the f32 C restatement: the parity checker)


def gather_bytes(b: bytes) -> list[bytes]:
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, b)
    return out


def main() -> int:
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    def new_uid() -> bytes:
        """A fresh NCCL unique id per communicator, broadcast from rank 0."""
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(bl.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        return bytes(uid.cpu().numpy().tobytes())

    failures = []

    def check(cond, what):
        if not cond:
            failures.append(what)

    transports = sys.argv[1:] or ["p2p", "nccl"]
    # ---- 1. compressed_allreduce API: real vs sim --------------------------
    for tp, d in [(tp, d) for tp in transports for d in (37, 10001, 4096 * 5 + 3, 1_000_003)]:
        cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=new_uid(),
                           transport=tp)
        check(cl.transport == tp, f"transport {cl.transport} != {tp}")
        sim = bl.SimCluster(world, d, device=local) if rank == 0 else None
        rng = np.random.default_rng(d)
        for step in range(3):
            x = rng.standard_normal((world, d)).astype(np.float32)
            es = 1.0 if step < 2 else 0.6
            out = cl.compressed_allreduce(x[rank], error_scale=es)
            outs = gather_bytes(out.tobytes())
            pk = gather_bytes(b"".join(cl.packet(rank, j) for j in range(world)))
            sp = gather_bytes(cl.server_packet(rank))
            we = gather_bytes(cl.worker_error(rank).tobytes())
            se = gather_bytes(cl.server_error(rank).tobytes())
            if rank == 0:
                ref = sim.compressed_allreduce(x, error_scale=es)
                for r in range(world):
                    check(outs[r] == ref.tobytes(), f"{tp} d={d} step={step} result rank {r}")
                    check(pk[r] == b"".join(sim.packet(r, j) for j in range(world)),
                          f"d={d} step={step} worker packets rank {r}")
                    check(sp[r] == sim.server_packet(r), f"d={d} step={step} server packet {r}")
                    check(we[r] == sim.worker_error(r).tobytes(), f"d={d} step={step} werr {r}")
                    check(se[r] == sim.server_error(r).tobytes(), f"d={d} step={step} serr {r}")
        led = cl.ledger()
        if rank == 0:
            check(led == sim.ledger(), f"d={d} ledger")
        for rep in range(3):  # several epochs of the lossless exchange
            x = rng.standard_normal((world, d)).astype(np.float32)
            lo = cl.lossless_allreduce(x[rank])
            los = gather_bytes(lo.tobytes())
            if rank == 0:
                ref = sim.lossless_allreduce(x)
                check(all(b == ref.tobytes() for b in los), f"{tp} d={d} lossless rep {rep}")
        cl.close()
        if sim:
            sim.close()

    # ---- 1b. endpoint statistics and verify_compensation -------------------
    # comm_sim.cpp:108-118,175-180: rank r refreshes its own endpoints
    # (worker r, server r); they must equal the simulated cluster's.
    for tp in transports:
        d = 50_001
        cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=new_uid(),
                           transport=tp, endpoint_stats=True, verify_compensation=True,
                           compensation_tolerance=2.0 ** -20)
        sim = bl.SimCluster(world, d, device=local, endpoint_stats=True) if rank == 0 else None
        rng = np.random.default_rng(11)
        for step in range(3):
            x = rng.standard_normal((world, d)).astype(np.float32)
            cl.compressed_allreduce(x[rank])
            ws, ss = cl.worker_stats()[rank], cl.server_stats()[rank]
            mine = np.array([ws.delta_l2, ws.delta_linf, ws.corrected_linf, ws.max_delta_linf,
                             ws.max_corrected_linf, ss.delta_l2, ss.delta_linf, ss.corrected_linf,
                             ss.max_delta_linf, ss.max_corrected_linf])
            allst = gather_bytes(mine.tobytes())
            if rank == 0:
                sim.compressed_allreduce(x)
                for r in range(world):
                    w2, s2 = sim.worker_stats()[r], sim.server_stats()[r]
                    ref = np.array([w2.delta_l2, w2.delta_linf, w2.corrected_linf, w2.max_delta_linf,
                                    w2.max_corrected_linf, s2.delta_l2, s2.delta_linf, s2.corrected_linf,
                                    s2.max_delta_linf, s2.max_corrected_linf])
                    check(allst[r] == ref.tobytes(), f"{tp} endpoint stats rank {r} step {step}")
        check(cl.compensation_checks() == 3 * (world + 1), f"{tp} compensation checks {cl.compensation_checks()}")
        cl.close()
        if sim:
            sim.close()

    # ---- 2. optimizer: warmup + freeze + compression stage -----------------
    for tp in transports:
        optimizer_check(rank, world, local, new_uid, check, tp)

    # ---- 3. strict mode and fail-stop (transactional steps) ----------------
    for tp in transports:
        strict_check(rank, world, local, new_uid, check, tp)
    if "p2p" in transports:
        failstop_check(rank, world, local, new_uid, check, "p2p")

    ok = torch.tensor([0 if failures else 1], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(("MULTIGPU PASS" if ok.item() else "MULTIGPU FAIL") + f" world={world} "
              f"transports={transports}", flush=True)
    if failures:
        print(f"rank {rank} failures: {failures[:10]}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok.item() else 1


def optimizer_check(rank, world, local, new_uid, check, tp):
    sizes = [3000, 2, 1024, 1023, 5000, 3, 4096 * 3 + 17, 77777]
    d = sum(sizes)
    steps, warm = 16, 5
    hp = bl.HyperParams(total_steps=steps, warmup_steps=warm, weight_decay=0.01,
                        scaled_error_feedback=True)
    cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=new_uid(),
                       transport=tp)
    opt = bl.Optimizer("onebit_lamb", sizes, hp, cl)
    if rank == 0:
        sim = bl.SimCluster(world, d, device=local)
        sopt = bl.Optimizer("onebit_lamb", sizes, hp, sim)
        # and the f32 oracle directly (not only transitively through SIM mode)
        ocl = O.Cluster("f32", world, d)
        oopt = O.Optimizer("f32", "onebit_lamb", sizes,
                           O.HyperParams(total_steps=steps, warmup_steps=warm, weight_decay=0.01,
                                         scaled_error_feedback=True))
    rng = np.random.default_rng(7)
    x0 = (rng.standard_normal(d) * 0.02).astype(np.float32)
    opt.set("x", x0)
    if rank == 0:
        sopt.set("x", x0)
        oopt.set("x", x0)
    sig = np.repeat(10.0 ** (-4 + 2 * rng.random(len(sizes))), sizes).astype(np.float32)
    for t in range(steps):
        g = (rng.standard_normal((world, d)) * sig).astype(np.float32)
        tr = opt.step(g[rank:rank + 1], t, 1e-3)
        xs = gather_bytes(opt.get("x").tobytes())
        trs = gather_bytes(tr.c.tobytes() + tr.r.tobytes() + tr.v_norm.tobytes())
        if rank == 0:
            st = sopt.step(g, t, 1e-3)
            ref_x = sopt.get("x").tobytes()
            ost = oopt.step(g, t, 1e-3, ocl)
            check(oopt.get("x").tobytes() == ref_x, f"{tp} oracle x t={t}")
            check(np.array_equal(np.asarray(ost["c"]), np.asarray(st.c)), f"{tp} oracle trace c t={t}")
            for r in range(world):
                check(xs[r] == ref_x, f"{tp} optimizer x rank {r} t={t}")
                check(trs[r] == st.c.tobytes() + st.r.tobytes() + st.v_norm.tobytes(),
                      f"optimizer trace rank {r} t={t}")
        if t == 2:  # mid-warmup read of the owner-sharded m and v (collective)
            for k in ("m", "v"):
                vals = gather_bytes(opt.get(k).tobytes())
                if rank == 0:
                    ref = sopt.get(k).tobytes()
                    check(all(v == ref for v in vals), f"{tp} optimizer mid-warmup {k}")
    for k in ("m", "v", "v_frozen"):
        vals = gather_bytes(opt.get(k).tobytes())
        if rank == 0:
            ref = sopt.get(k).tobytes()
            check(all(v == ref for v in vals), f"{tp} optimizer {k}")
            check(oopt.get(k).tobytes() == ref, f"{tp} oracle {k}")
    opt.close()
    cl.close()

    # check_gradients (optimizers.cpp:99-117) in the multi-process warmup: a
    # non-finite element of the last rank's gradient lying in chunk 0 is read
    # by rank 0 (over NVLink in P2P mode) and forwarded to every rank, so every
    # rank raises the reference's message (fused mode: after the step).
    cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=new_uid(),
                       transport=tp)
    opt = bl.Optimizer("onebit_lamb", sizes, hp, cl)
    for t in range(3):
        g = (rng.standard_normal((1, d)) * sig).astype(np.float32)
        bad = t == 2 and rank == world - 1
        if bad:
            g[0, 5] = np.nan
        try:
            opt.step(g, t, 1e-3)
            raised = ""
        except Exception as exc:  # noqa: BLE001 - the message is checked below
            raised = str(exc)
        if t == 2:  # every rank, on both transports
            check("non-finite gradient" in raised and f"worker {world - 1}" in raised,
                  f"{tp} rank {rank}: non-finite gradient not reported: {raised!r}")
        else:
            check(raised == "", f"{tp} rank {rank} t={t} unexpected error {raised!r}")
    opt.close()
    cl.close()

    # ... and in the compression stage (K1's fused check), after a one-step warmup.
    cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=new_uid(),
                       transport=tp)
    opt = bl.Optimizer("onebit_lamb", sizes, bl.HyperParams(total_steps=4, warmup_steps=1), cl)
    for t in range(3):
        g = (rng.standard_normal((1, d)) * sig).astype(np.float32)
        if t == 2 and rank == world - 1:
            g[0, d - 7] = np.inf
        try:
            opt.step(g, t, 1e-3)
            raised = ""
        except Exception as exc:  # noqa: BLE001 - the message is checked below
            raised = str(exc)
        if t == 2:
            check("non-finite gradient" in raised and f"worker {world - 1}" in raised,
                  f"{tp} rank {rank}: compression-stage non-finite gradient not reported: {raised!r}")
        else:
            check(raised == "", f"{tp} rank {rank} t={t} unexpected error {raised!r}")
    opt.close()
    cl.close()


def state_bytes(opt, cl, rank):
    return b"".join(opt.get(k).tobytes() for k in ("x", "m", "v", "v_frozen")) + \
        cl.worker_error(rank).tobytes() + cl.server_error(rank).tobytes() + cl.server_packet(rank)


def strict_check(rank, world, local, new_uid, check, tp):
    """Strict mode (optimizers.cpp:99-117,337): a non-finite element in the
    last rank's gradient, in the warmup stage and in the compression stage,
    raises the reference's message on EVERY rank before anything changed; the
    run then continues bit-identically to a simulated cluster that never saw
    the bad steps."""
    sizes = [3000, 2, 1024, 1023, 5000, 3, 4096 * 3 + 17, 77777]
    names = [f"layer.{i}" for i in range(len(sizes))]
    layout = list(zip(names, sizes))
    d = sum(sizes)
    steps, warm = 10, 4
    hp = bl.HyperParams(total_steps=steps + 2, warmup_steps=warm)
    cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=new_uid(), transport=tp)
    opt = bl.Optimizer("onebit_lamb", layout, hp, cl, strict=True)
    if rank == 0:
        sim = bl.SimCluster(world, d, device=local)
        sopt = bl.Optimizer("onebit_lamb", layout, hp, sim, strict=True)
    rng = np.random.default_rng(17)
    x0 = (rng.standard_normal(d) * 0.02).astype(np.float32)
    opt.set("x", x0)
    if rank == 0:
        sopt.set("x", x0)
    sig = np.repeat(10.0 ** (-4 + 2 * rng.random(len(sizes))), sizes).astype(np.float32)
    t = 0
    while t < steps:
        g = (rng.standard_normal((world, d)) * sig).astype(np.float32)
        for bad_t in (2, 6):  # one warmup-stage and one compression-stage rejection
            if t == bad_t:
                gb = g.copy()
                gb[world - 1, 3000 + 2 + 1024 + 17] = np.inf  # layer.3
                before = state_bytes(opt, cl, rank)
                try:
                    opt.step(gb[rank:rank + 1], t, 1e-3)
                    raised = ""
                except bl.NumericalError as exc:
                    raised = str(exc)
                want = f"non-finite gradient at step {t}, worker {world - 1}, layer 'layer.3'"
                check(raised == want, f"{tp} strict rank {rank} t={t}: {raised!r} != {want!r}")
                check(state_bytes(opt, cl, rank) == before, f"{tp} strict rank {rank} t={t}: state changed")
                if rank == 0:
                    try:
                        sopt.step(gb, t, 1e-3)
                        sraised = ""
                    except bl.NumericalError as exc:
                        sraised = str(exc)
                    check(sraised == want, f"sim strict t={t}: {sraised!r}")
        tr = opt.step(g[rank:rank + 1], t, 1e-3)
        xs = gather_bytes(opt.get("x").tobytes() + tr.c.tobytes())
        if rank == 0:
            st = sopt.step(g, t, 1e-3)
            ref = sopt.get("x").tobytes() + st.c.tobytes()
            for r in range(world):
                check(xs[r] == ref, f"{tp} strict: x rank {r} t={t} after the rejected steps")
        t += 1
    opt.close()
    cl.close()


def failstop_check(rank, world, local, new_uid, check, tp):
    """A rank late past the peer timeout (host stall before the step) aborts
    the step on EVERY rank before any state changed -- the late rank included
    -- instead of letting the others run on stale packets; the next step then
    proceeds normally and matches a simulated cluster that never saw it."""
    import time

    sizes = [3000, 2, 1024, 1023, 5000, 3, 4096 * 3 + 17, 77777]
    d = sum(sizes)
    hp = bl.HyperParams(total_steps=12, warmup_steps=2)
    cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=new_uid(), transport=tp)
    cl.set_peer_timeout(1500.0)
    opt = bl.Optimizer("onebit_lamb", sizes, hp, cl)
    if rank == 0:
        sim = bl.SimCluster(world, d, device=local)
        sopt = bl.Optimizer("onebit_lamb", sizes, hp, sim)
    rng = np.random.default_rng(23)
    x0 = (rng.standard_normal(d) * 0.02).astype(np.float32)
    opt.set("x", x0)
    if rank == 0:
        sopt.set("x", x0)
    sig = np.repeat(10.0 ** (-4 + 2 * rng.random(len(sizes))), sizes).astype(np.float32)
    for t in range(6):
        g = (rng.standard_normal((world, d)) * sig).astype(np.float32)
        for late_t in (1, 4):  # a late rank in the warmup stage and in the compression stage
            if t != late_t:
                continue
            before = state_bytes(opt, cl, rank)
            if rank == world - 1:
                time.sleep(4.0)  # > the 1.5 s timeout: the others give up
            t0 = time.time()
            try:
                opt.step(g[rank:rank + 1], t, 1e-3)
                raised = ""
            except bl.NcclError as exc:
                raised = str(exc)
            took = time.time() - t0
            check("aborted on every rank before any state changed" in raised,
                  f"{tp} failstop rank {rank} t={t}: {raised!r}")
            check(took < 30.0, f"{tp} failstop rank {rank} t={t}: took {took:.1f} s")
            check(state_bytes(opt, cl, rank) == before, f"{tp} failstop rank {rank} t={t}: state changed")
            dist.barrier()
        tr = opt.step(g[rank:rank + 1], t, 1e-3)
        xs = gather_bytes(opt.get("x").tobytes() + tr.c.tobytes())
        if rank == 0:
            st = sopt.step(g, t, 1e-3)
            ref = sopt.get("x").tobytes() + st.c.tobytes()
            for r in range(world):
                check(xs[r] == ref, f"{tp} failstop: x rank {r} t={t}")
    opt.close()
    cl.close()


if __name__ == "__main__":
    sys.exit(main())
