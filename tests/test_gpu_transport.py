"""Device transport semantics (reference tests/test_transport.py analogs) + the
notification happens-before stress (test_acceptance.py:124-222) on one GPU."""

import struct
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def make_world(size=2, seg=256, notif=16, inline=True):
    from paper_1706_00095_b200.transport import LocalWorld

    world = LocalWorld(size, inline=inline)
    trs = [world.transport(r) for r in range(size)]
    for tr in trs:
        tr.segment_create(0, seg, notif)
    return world, trs


def test_write_delivers_bytes_then_notification(cuda):
    from paper_1706_00095_b200.transport import WriteRequest

    world, (a, b) = make_world()
    payload = np.arange(4, dtype=np.float64)
    a.segment(0).write(0, payload.tobytes())
    t = a.write_notify(WriteRequest(0, 0, 1, 0, 64, 32, 5, 9))
    t.wait(1.0)
    assert b.notify_poll(0, 5, 1) == [(5, 9)]
    assert b.notify_poll(0, 1, 15) == [(5, 9)], "poll must not consume"
    assert b.segment(0).read(64, 32) == payload.tobytes()
    assert b.notify_reset(0, 5) == 9
    assert b.notify_reset(0, 5) == 0
    assert b.notify_poll(0, 0, 16) == []
    world.close()


def test_self_write_and_async_tickets(cuda):
    from paper_1706_00095_b200.transport import WriteRequest

    world, (a, b) = make_world(inline=False)
    a.segment(0).write(0, b"\xaa" * 8)
    t = a.write_notify(WriteRequest(0, 0, 0, 0, 128, 8, 3, 1))
    a.ticket_wait_all([t], timeout=5.0)
    assert t.done
    assert a.segment(0).read(128, 8) == b"\xaa" * 8
    assert a.notify_poll(0, 3, 1) == [(3, 1)]
    world.close()


def test_validation_errors(cuda):
    from paper_1706_00095_b200.errors import ConfigError, ProtocolError, RangeError, RoutingError
    from paper_1706_00095_b200.transport import WriteRequest

    world, (a, b) = make_world()
    with pytest.raises(ProtocolError):
        a.write_notify(WriteRequest(0, 0, 1, 0, 0, 8, 1, 0))
    with pytest.raises(RangeError):
        a.write_notify(WriteRequest(0, 250, 1, 0, 0, 8, 1, 1))
    with pytest.raises(RangeError):
        a.write_notify(WriteRequest(0, 0, 1, 0, 252, 8, 1, 1))
    with pytest.raises(RangeError):
        a.write_notify(WriteRequest(0, 0, 1, 0, 0, 8, 16, 1))
    with pytest.raises(RoutingError):
        a.write_notify(WriteRequest(0, 0, 7, 0, 0, 8, 1, 1))
    with pytest.raises(ConfigError):
        a.segment_create(0, 64, 1)
    with pytest.raises(ConfigError):
        a.segment_create(15, 64, 1)
    with pytest.raises(RangeError):
        b.notify_poll(0, 10, 10)
    world.close()


def test_chunked_write_ids_follow_the_layout_rule(cuda):
    """Final chunk carries the base id, earlier chunk j carries base+1+j (layout.py:130-139)."""
    world, (a, b) = make_world(seg=1000, notif=64)
    data = bytes(range(256)) * 3
    a.segment(0).write(0, data)
    a.write_notify_chunked(0, 0, 1, 0, 100, 700, 64, 20, 3)
    n = -(-700 // 64)
    ids = [nid for nid, v in b.notify_poll(0, 0, 64)]
    assert ids == sorted([20] + [21 + j for j in range(n - 1)])
    assert b.segment(0).read(100, 700) == data[:700]
    world.close()


def test_zero_byte_notify(cuda):
    from paper_1706_00095_b200.transport import WriteRequest

    world, (a, b) = make_world()
    a.write_notify(WriteRequest(0, 0, 1, 0, 0, 0, 2, 4))
    assert b.notify_poll(0, 2, 1) == [(2, 4)]
    world.close()


def test_happens_before_stress(cuda):
    """Randomised notify-writes 1 B..1 MiB with a CRC trailer: when the notification is
    visible the payload must be complete (criterion 3, test_acceptance.py:124-222)."""
    from paper_1706_00095_b200.transport import WriteRequest

    trials, maxp = 2000, 1 << 20
    world, (a, b) = make_world(seg=maxp + 64, notif=16, inline=False)
    rng = np.random.default_rng(101)
    sizes = np.clip((2.0 ** rng.uniform(0, 20, trials)).astype(np.int64), 1, maxp)
    sizes[0], sizes[1] = 1, maxp
    pool = torch.from_numpy(rng.integers(0, 256, size=maxp + 4096, dtype=np.uint8)).cuda()
    src = a.segment(0).data
    dst = b.segment(0).data
    corrupt = 0
    for t in range(trials):
        n = int(sizes[t])
        off = int(rng.integers(0, 4096))
        body = pool[off:off + n]
        crc = zlib.crc32(body.cpu().numpy().tobytes())
        with torch.cuda.stream(a.stream):
            src[:n].copy_(body)
            src[n:n + 4].copy_(torch.frombuffer(bytearray(struct.pack("<I", crc)), dtype=torch.uint8).cuda())
        nid, value = t % 8 + 1, t % 60000 + 1
        tk = a.write_notify(WriteRequest(0, 0, 1, 0, 0, n + 4, nid, value))
        while True:  # poll from the host while the write may still be in flight
            hits = b.notify_poll(0, nid, 1)
            if hits:
                break
        assert hits == [(nid, value)]
        got = dst[:n + 4].cpu().numpy().tobytes()
        if zlib.crc32(got[:n]) != struct.unpack("<I", got[n:n + 4])[0]:
            corrupt += 1
        b.notify_reset(0, nid)
        tk.wait(5.0)
    world.close()
    assert corrupt == 0
