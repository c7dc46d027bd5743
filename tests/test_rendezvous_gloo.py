"""N>1 host logic on CPU: the segment-handle rendezvous over a world_size-2 gloo group."""

import os

import pytest
import torch.multiprocessing as mp


def _worker(rank, world, port, q, mismatch):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1706_00095_b200.errors import ConfigError
    from paper_1706_00095_b200.rendezvous import exchange

    mine = {0: (bytes([rank]) * 64, 100 + rank, 7), 15: (bytes([9]) * 64, 256, 8)}
    if mismatch and rank == 1:
        mine[3] = (b"\0" * 64, 1, 1)
    try:
        every = exchange(mine, rank, world, None)
        q.put((rank, "ok", [sorted(e) for e in every], [e[0][1] for e in every]))
    except ConfigError as exc:
        q.put((rank, "config", str(exc), None))
    dist.destroy_process_group()


def _run(mismatch):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, mismatch)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(out)


def test_handles_reach_every_rank():
    out = _run(False)
    for rank, status, ids, sizes in out:
        assert status == "ok"
        assert ids == [[0, 15], [0, 15]]
        assert sizes == [100, 101]


def test_mismatched_segment_sets_are_rejected():
    out = _run(True)
    assert all(status == "config" for _, status, _, _ in out)
