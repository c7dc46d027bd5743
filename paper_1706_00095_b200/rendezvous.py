"""One-time exchange of segment handles between ranks (plumbing, not the data path).

Each rank contributes {segment_id: (ipc_handle_bytes, size, notification_count)};
every rank receives the list indexed by rank.  Uses torch.distributed object
collectives on whatever group the caller initialised (gloo is enough), which is
also how the CPU tests exercise the N>1 host logic without a GPU.
"""

from __future__ import annotations

from .errors import ConfigError, RoutingError


def exchange(mine: dict, rank: int, world_size: int, group=None) -> list:
    import torch.distributed as dist

    if world_size == 1:
        return [mine]
    if not dist.is_available() or not dist.is_initialized():
        raise ConfigError("multi-rank rendezvous needs an initialised torch.distributed group")
    if dist.get_world_size(group) != world_size or dist.get_rank(group) != rank:
        raise RoutingError(
            f"process group (rank {dist.get_rank(group)}/{dist.get_world_size(group)}) does not match "
            f"transport rank {rank}/{world_size}")
    every: list = [None] * world_size
    dist.all_gather_object(every, mine, group=group)
    ids = set(mine)
    for peer, segs in enumerate(every):
        if set(segs) != ids:
            raise ConfigError(f"rank {peer} registered segments {sorted(segs)}, rank {rank} has {sorted(ids)}")
    return every
