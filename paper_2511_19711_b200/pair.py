"""Party-pair bootstrap for MPC_MODE_PAIR: ranks (2k, 2k+1) form a pair,
rank 2k is party 0.  The two contexts swap their exchange-memory handles over
torch.distributed (any backend: the handle is 64 opaque bytes) and map each other's
receive buffers; after that every opening travels through NVLink peer memory inside
the fused kernels, with no collective on the data path."""
from __future__ import annotations

import torch
import torch.distributed as dist


def pair_layout(rank: int, world: int):
    """-> (party, peer_rank, pair_index, n_pairs) for rank in a world of even size."""
    if world % 2:
        raise ValueError("PAIR mode needs an even number of ranks (party 0 / party 1 per pair)")
    return rank % 2, rank ^ 1, rank // 2, world // 2


def exchange_handles(handle: bytes, group=None) -> bytes:
    """All-gather the 64-byte handles and return the peer's (rank ^ 1)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = torch.frombuffer(bytearray(handle), dtype=torch.uint8)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = mine.to(dev)
    out = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(out, mine, group=group)
    _, peer, _, _ = pair_layout(rank, world)
    return bytes(out[peer].cpu().numpy().tobytes())


def connect(ctx, group=None):
    """Export this party's exchange memory, receive the peer's and map it."""
    peer = exchange_handles(ctx.pair_export(), group)
    ctx.pair_connect(peer)
    dist.barrier(group)
    return ctx
