"""Memory-ordering stress across real GPUs (NVLink, CUDA IPC), SURVEY §5 / §8 a13.

1. The reference's notification happens-before criterion (tests/test_acceptance.py:124-222,
   `_STRESS_TRIALS = 10_000` at :127): 10^4 notify-writes of 1 B .. 1 MiB at random
   offsets from GPU 0 into GPU 1's segment, each payload followed by its CRC32; GPU 1's
   host polls the notification while the write may still be in flight and, once it is
   visible, the payload must be complete.  An ack notification (zero-byte write back)
   lets the writer reuse its buffers.
2. The fence-free protocols under concurrent folds: many iterations of the exchange with
   the LL (8-byte {value, epoch} words) and L128 (128-byte lines, flag in the line)
   one-shots and the TMA bulk two-shot, every iteration's gradients fresh, both ranks
   folding while the peer writes; one torn word/line or early read anywhere would leave
   the weights different from the oracle's (fast32 weights + momentum carry every error
   forward), so the final comparison covers every iteration.

Skipped unless >= 2 GPUs are visible (the driver's 1-GPU suite does not run them; their
logs are committed under profiles/).
"""

import os
import struct
import zlib

import numpy as np
import pytest
import torch

from test_gpu_multi import _ngpu, _spawn

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

TRIALS = 10_000
MAXP = 1 << 20


def _crc_worker(rank, world, port, trials, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    from paper_1706_00095_b200.transport import DistTransport, WriteRequest

    try:
        tr = DistTransport(rank, world, rank, timeout_s=30.0)
        tr.segment_create(0, MAXP + 4096 + 64, 16)
        tr.barrier()
        rng = np.random.default_rng(2024)  # same stream on both ranks: sizes and offsets agree
        sizes = np.clip((2.0 ** rng.uniform(0, 20, trials)).astype(np.int64), 1, MAXP)
        sizes[0], sizes[1] = 1, MAXP
        offs = rng.integers(0, 4096, trials)
        pool = torch.from_numpy(np.random.default_rng(7).integers(0, 256, size=MAXP + 4096, dtype=np.uint8)).cuda()
        seg = tr.segment(0).data
        corrupt, early = 0, 0
        for t in range(trials):
            n, off = int(sizes[t]), int(offs[t])
            nid, value = t % 8 + 1, t // 8 + 1
            if rank == 0:
                body = pool[off:off + n]
                crc = zlib.crc32(body.cpu().numpy().tobytes())
                with torch.cuda.stream(tr.stream):
                    seg[off:off + n].copy_(body)
                    seg[off + n:off + n + 4].copy_(
                        torch.frombuffer(bytearray(struct.pack("<I", crc)), dtype=torch.uint8).cuda())
                tk = tr.write_notify(WriteRequest(0, off, 1, 0, off, n + 4, nid, value))
                while not tr.notify_poll(0, 9, 1):  # wait for rank 1's ack before reusing buffers
                    pass
                tr.notify_reset(0, 9)
                tk.wait(10.0)
            else:
                while True:  # poll while the write may still be in flight
                    hits = tr.notify_poll(0, nid, 1)
                    if hits:
                        break
                if hits != [(nid, value)]:
                    early += 1
                got = seg[off:off + n + 4].cpu().numpy().tobytes()
                if zlib.crc32(got[:n]) != struct.unpack("<I", got[n:n + 4])[0]:
                    corrupt += 1
                tr.notify_reset(0, nid)
                tr.write_notify(WriteRequest(0, 0, 0, 0, 0, 0, 9, t + 1))  # ack (zero-byte notify)
        torch.cuda.synchronize()
        q.put((rank, (corrupt, early), tr.device_status()))
        tr.close()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc(), -1))
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_happens_before_stress_across_gpus():
    out = _spawn(_crc_worker, 2, TRIALS)
    for rank, res, status in out:
        assert status == 0 and res == (0, 0), (rank, res, status)


def _fold_stress_worker(rank, world, port, variant, iters, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    from oracle import pipesgd_oracle as O
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import DistTransport

    try:
        tr = DistTransport(rank, world, rank, timeout_s=30.0)
        # sizes across the protocols' regimes: sub-line, ragged lines / words, many chunks
        elems = [7, 4099, 65536, 1 << 18, (1 << 20) + 5] if variant != "twoshot_bulk" else \
            [4099, 1 << 18, (1 << 22) + 12, 3 << 20]
        hyper = dict(lr=0.01, momentum=0.9, weight_decay=5e-4)
        x = DeviceExchange(tr, elems, mode="fast32", variant=variant, chunk_elems=16384,
                           flags=("allow_l128",) if "l128" in variant else (), **hyper)
        w = [O.seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)).astype(np.float32) for l, n in enumerate(elems)]
        v = [np.zeros(n, np.float32) for n in elems]
        for l in range(len(elems)):
            x.layer_views[l].copy_(torch.from_numpy(w[l]))
        torch.cuda.synchronize()
        tr.barrier()
        x.connect()
        comp = torch.cuda.current_stream()
        for k in range(iters):
            grads = {}
            for l in range(len(elems)):
                if k:
                    x.gate(l, k - 1)  # the next forward waits only for this layer
            for l in reversed(range(len(elems))):
                n = elems[l]
                gs = [np.random.default_rng([r, l, k]).standard_normal(n, dtype=np.float32) * np.float32(1e-2)
                      for r in range(world)]
                grads[l] = gs
                g = torch.from_numpy(gs[rank]).cuda()
                x.stream.wait_stream(comp)
                g.record_stream(x.stream)
                x.launch(l, k, [g])
            for l in range(len(elems)):
                w[l], v[l] = O.exchange_iteration(grads[l], w[l], 0.01, "fast32", state=v[l], scale=1.0 / world,
                                                  momentum=0.9, weight_decay=5e-4)
        for l in range(len(elems)):
            x.gate(l, iters - 1)
        torch.cuda.synchronize()
        bad = [l for l in range(len(elems)) if x.layer_views[l].cpu().numpy().tobytes() != w[l].tobytes()]
        q.put((rank, bad, tr.device_status()))
        x.close()
        tr.close()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc(), -1))
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("variant", ["oneshot_ll", "oneshot_l128", "twoshot_bulk", "twoshot", "twoshot_l128"])
def test_concurrent_fold_stress(variant):
    """Hundreds of back-to-back iterations, no host synchronisation between them (only
    the per-layer gates), fresh gradients each: bit-exact with the oracle at the end."""
    out = _spawn(_fold_stress_worker, _ngpu(), variant, 200)
    for rank, bad, status in out:
        assert bad == [] and status == 0, (rank, bad, status)
