"""Host plumbing for the one-process-per-GPU (NCCL mode) cluster.

torch.distributed is used only as the launcher's rendezvous: it carries the
128-byte NCCL unique id from rank 0 to every rank and reduces timings.  The
packet exchange itself runs inside libbitlamb_b200.so on the library's own
NCCL communicator (include/bitlamb_b200.h, BL_MODE_NCCL).
"""
from __future__ import annotations

import os


def env_rank() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload: bytes | None, nbytes: int, src: int = 0) -> bytes:
    """Broadcast `payload` (only needed on `src`) over the default process group."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    if dist.get_rank() == src:
        assert payload is not None and len(payload) == nbytes
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())


def new_unique_id(generate=None) -> bytes:
    """A fresh NCCL unique id for one communicator, made on rank 0 and
    broadcast (ncclGetUniqueId, via bl_nccl_get_unique_id)."""
    import torch.distributed as dist

    if generate is None:
        from . import bitlamb

        generate = bitlamb.nccl_unique_id
    return broadcast_bytes(generate() if dist.get_rank() == 0 else None, 128)


def max_over_ranks(value: float) -> float:
    """Max of a per-rank timing (the driver's multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def chunk_bounds(dim: int, world: int, rank: int) -> tuple[int, int]:
    """Global range [begin, end) of the chunk rank serves (comm_sim.cpp:58-59:
    P = ceil(dim/n)*n, c = P/n; the tail beyond dim is zero padding)."""
    padded = -(-dim // world) * world
    c = padded // world
    return rank * c, (rank + 1) * c


def packet_bytes(chunk: int) -> int:
    """serialize() size of one chunk message (compression.cpp:91-99)."""
    return (chunk + 7) // 8 + 4
