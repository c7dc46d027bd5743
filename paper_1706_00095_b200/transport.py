"""One-sided notify-write transport over CUDA peer memory (the drop-in boundary).

Mirrors the reference transport ABI (transport/base.py:170-225, inproc.py:129-149):
`segment_create`, `segment`, `write_notify(WriteRequest) -> Ticket`, `notify_poll`,
`notify_reset`, `ticket_wait_all`, `barrier`, `close`, and the attributes `rank`,
`world_size`, `barrier_calls`.  Underneath, every call goes through libpgx.so:

* a Segment is device memory ([data | u32 notification flags]) owned by the C
  library; Python sees aliasing torch views (like ``Segment.view_f64``);
* ``write_notify`` enqueues a kernel on this rank's CUDA stream that stores the
  payload straight into the peer's segment (NVLink peer stores when the peer is
  another GPU) and then raises the notification with a system-scope release;
* a Ticket is a CUDA event recorded after that kernel.

Two worlds:

* :class:`LocalWorld` — several ranks on ONE GPU inside one process (the analog
  of ``InprocWorld``, inproc.py:62-127), host barrier, for protocol tests.  With
  ``inline=True`` a write is complete when ``write_notify`` returns, like the
  reference's zero-latency inline delivery (inproc.py:137-139).
* :class:`DistTransport` — one process per GPU; segments are exported with CUDA
  IPC and attached by every peer during the first ``barrier()`` (the rendezvous
  the reference does before its loop, runtime.py:311-319).
"""

from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ConfigError, ProtocolError, RangeError, TransportError

CONTROL_SEGMENT = _lib.CONTROL_SEGMENT


@dataclass(frozen=True)
class LatencyModel:
    """Accepted for API compatibility (base.py:25-36); only zero latency is meaningful
    on real hardware, so nonzero values are rejected."""

    fixed_ns: int = 0
    per_byte_ns: float = 0.0

    @property
    def is_zero(self) -> bool:
        return self.fixed_ns == 0 and self.per_byte_ns == 0.0


@dataclass(frozen=True)
class WriteRequest:
    """One one-sided write (base.py:40-55); the source range must stay unmodified
    until the ticket completes; notification_value must be nonzero."""

    local_segment: int
    local_offset: int
    rank: int
    remote_segment: int
    remote_offset: int
    size: int
    notification_id: int
    notification_value: int


class Ticket:
    """Completion handle of one write: a CUDA event (base.py:58-91)."""

    __slots__ = ("_ev", "error", "completed_at_ns")

    def __init__(self, event_handle=None):
        self._ev = event_handle
        self.error = None
        self.completed_at_ns = 0 if event_handle else time.monotonic_ns()

    @property
    def done(self) -> bool:
        if self._ev is None:
            return True
        rc = _lib.lib().pgx_ticket_query(self._ev)
        if rc < 0:
            self.error = TransportError(_lib.last_error())
            return True
        if rc == 1:
            self._finish()
            return True
        return False

    def _finish(self):
        if self._ev is not None:
            _lib.lib().pgx_ticket_release(self._ev)
            self._ev = None
            self.completed_at_ns = time.monotonic_ns()

    def wait(self, timeout: float | None = None) -> None:
        if self.error is not None:
            raise TransportError(str(self.error))
        if self._ev is None:
            return
        rc = _lib.lib().pgx_ticket_wait(self._ev, -1.0 if timeout is None else float(timeout))
        if rc != 0:
            msg = _lib.last_error()
            raise TransportError(msg.replace("write did not complete", "write did not complete") or "write failed")
        self._finish()

    def __del__(self):
        try:
            if self._ev is not None:
                _lib.lib().pgx_ticket_release(self._ev)
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


def completed_ticket() -> Ticket:
    return Ticket(None)


class _CudaArray:
    """__cuda_array_interface__ wrapper so torch can alias library-owned memory."""

    def __init__(self, ptr: int, nbytes: int, owner):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3, "strides": None,
        }
        self._owner = owner


class Segment:
    """Remotely writable device bytes plus notification slots (base.py:129-167)."""

    def __init__(self, transport, segment_id: int, data_ptr: int, flags_ptr: int, size: int, count: int):
        self.segment_id = segment_id
        self.size = size
        self.notification_count = count
        self.data_ptr = data_ptr
        self.flags_ptr = flags_ptr
        self._tr = transport
        self.data = torch.as_tensor(_CudaArray(data_ptr, size, self), device=transport.device)

    def check_range(self, offset: int, size: int) -> None:
        if offset < 0 or size < 0 or offset + size > self.size:
            raise RangeError(f"range [{offset}, {offset + size}) outside segment {self.segment_id} of size {self.size}")

    def view(self, dtype: torch.dtype, offset: int, count: int) -> torch.Tensor:
        eb = torch.empty((), dtype=dtype).element_size()
        self.check_range(offset, count * eb)
        if offset % eb:
            raise RangeError(f"{dtype} view needs {eb}-byte alignment, offset {offset}")
        return self.data[offset: offset + count * eb].view(dtype)

    def view_f64(self, offset: int, count: int) -> torch.Tensor:
        return self.view(torch.float64, offset, count)

    def view_f32(self, offset: int, count: int) -> torch.Tensor:
        return self.view(torch.float32, offset, count)

    def write(self, offset: int, payload) -> None:
        """Host bytes -> segment (synchronous on the rank's stream)."""
        n = len(payload)
        self.check_range(offset, n)
        if n:
            src = torch.frombuffer(bytearray(payload), dtype=torch.uint8)
            with torch.cuda.stream(self._tr.stream):
                self.data[offset:offset + n].copy_(src, non_blocking=False)
            self._tr.stream.synchronize()

    def read(self, offset: int, size: int) -> bytes:
        self.check_range(offset, size)
        self._tr.stream.synchronize()
        return bytes(self.data[offset:offset + size].cpu().numpy().tobytes())


class CudaTransport:
    """Per-rank transport over a libpgx world (TransportBase analog, base.py:170-225)."""

    inline = False

    def __init__(self, rank: int, world_size: int, device: int = 0, latency: LatencyModel | None = None):
        if world_size < 1:
            raise ConfigError(f"world size must be >= 1, got {world_size}")
        if not (0 <= rank < world_size):
            raise ConfigError(f"rank {rank} outside world of size {world_size}")
        if latency is not None and not latency.is_zero:
            raise ConfigError("latency injection is a CPU-desk device; real links have real latency")
        self.rank = rank
        self.world_size = world_size
        self.device = torch.device("cuda", device)
        self.latency = latency or LatencyModel()
        self.barrier_calls = 0
        self._segments: dict[int, Segment] = {}
        self._peer_segments: dict[tuple[int, int], Segment] = {}
        h = C.c_void_p()
        _lib.call("pgx_world_create", rank, world_size, device, C.byref(h))
        self.handle = h
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(device=self.device)
        self._closed = False

    # -- segments -------------------------------------------------------------
    def segment_create(self, segment_id: int, size: int, notification_count: int) -> Segment:
        if not (0 <= segment_id < 65536):
            raise ConfigError(f"segment id {segment_id} outside u16 range")
        if segment_id == CONTROL_SEGMENT:
            raise ConfigError(f"segment id {CONTROL_SEGMENT} is reserved for the transport")
        if segment_id in self._segments:
            raise ConfigError(f"segment {segment_id} already exists on rank {self.rank}")
        d, f = C.c_void_p(), C.c_void_p()
        _lib.call("pgx_segment_create", self.handle, segment_id, size, notification_count, C.byref(d), C.byref(f))
        seg = Segment(self, segment_id, d.value, f.value, size, notification_count)
        self._segments[segment_id] = seg
        self._on_segment_created(seg)
        return seg

    def adopt_segment(self, segment_id: int) -> Segment:
        """Register a segment the C library created in this world (device exchange)."""
        d, f, sz, cnt = C.c_void_p(), C.c_void_p(), C.c_uint64(), C.c_uint32()
        _lib.call("pgx_segment_info", self.handle, self.rank, segment_id, C.byref(d), C.byref(f), C.byref(sz),
                  C.byref(cnt))
        seg = Segment(self, segment_id, d.value, f.value, sz.value, cnt.value)
        self._segments[segment_id] = seg
        self._on_segment_created(seg)
        return seg

    def _on_segment_created(self, seg: Segment) -> None:
        pass

    def segment(self, segment_id: int) -> Segment:
        try:
            return self._segments[segment_id]
        except KeyError:
            raise ConfigError(f"segment {segment_id} does not exist on rank {self.rank}") from None

    # -- local notification ops (base.py:203-208) --------------------------------
    def notify_poll(self, segment_id: int, first_id: int, count: int) -> list[tuple[int, int]]:
        seg = self.segment(segment_id)
        if first_id < 0 or count < 0 or first_id + count > seg.notification_count:
            raise RangeError(f"poll range [{first_id}, {first_id + count}) outside 0..{seg.notification_count - 1}")
        if count == 0:
            return []
        ids = (C.c_uint32 * count)()
        vals = (C.c_uint32 * count)()
        n = C.c_uint32()
        _lib.call("pgx_notify_poll", self.handle, segment_id, first_id, count, ids, vals, count, C.byref(n))
        return [(ids[i], vals[i]) for i in range(n.value)]

    def notify_reset(self, segment_id: int, notification_id: int) -> int:
        self.segment(segment_id)
        old = C.c_uint32()
        _lib.call("pgx_notify_reset", self.handle, segment_id, notification_id, C.byref(old))
        return old.value

    # -- writes ---------------------------------------------------------------------
    def _validate(self, req: WriteRequest) -> None:
        if req.size < 0:
            raise RangeError(f"write size must be >= 0, got {req.size}")
        if req.notification_value == 0:
            raise ProtocolError("notification value 0 is reserved; use values >= 1")
        self.segment(req.local_segment).check_range(req.local_offset, req.size)

    def write_notify(self, req: WriteRequest) -> Ticket:
        self._validate(req)
        self._ensure_connected(req.rank)
        _lib.call("pgx_write_notify", self.handle, req.local_segment, req.local_offset, req.rank,
                  req.remote_segment, req.remote_offset, req.size, req.notification_id,
                  req.notification_value, self.stream.cuda_stream)
        return self._ticket()

    def write_notify_chunked(self, local_segment, local_offset, rank, remote_segment, remote_offset, size,
                             chunk_bytes, base_id, value) -> Ticket:
        """All chunks of one RankBase._send transfer (runtime.py:185-224) in one launch."""
        if value == 0:
            raise ProtocolError("notification value 0 is reserved; use values >= 1")
        self._ensure_connected(rank)
        _lib.call("pgx_write_notify_chunked", self.handle, local_segment, local_offset, rank, remote_segment,
                  remote_offset, size, chunk_bytes, base_id, value, self.stream.cuda_stream)
        return self._ticket()

    def _ticket(self) -> Ticket:
        if self.inline:
            self.stream.synchronize()
            return completed_ticket()
        ev = C.c_void_p()
        _lib.call("pgx_ticket_record", self.stream.cuda_stream, C.byref(ev))
        return Ticket(ev.value)

    def _ensure_connected(self, rank: int) -> None:
        pass

    def ticket_wait_all(self, tickets, timeout: float | None = None) -> None:
        deadline = None if timeout is None else time.monotonic() + timeout
        for t in tickets:
            remaining = None if deadline is None else max(0.0, deadline - time.monotonic())
            t.wait(remaining)

    # -- status ----------------------------------------------------------------------
    def device_status(self) -> int:
        s = C.c_uint32()
        _lib.call("pgx_world_status", self.handle, C.byref(s))
        return s.value

    def close(self) -> None:
        if not self._closed:
            self._closed = True
            self.stream.synchronize()
            _lib.call("pgx_world_destroy", self.handle)


class LocalTransport(CudaTransport):
    def __init__(self, world: "LocalWorld", rank: int):
        self._world = world
        self.inline = world.inline
        super().__init__(rank, world.world_size, world.device_of(rank))

    def _on_segment_created(self, seg: Segment) -> None:
        self._world._publish(self.rank, seg)

    def barrier(self) -> None:
        self.barrier_calls += 1
        self.stream.synchronize()
        try:
            self._world._barrier.wait()
        except threading.BrokenBarrierError as exc:
            raise TransportError("barrier broken; a peer failed") from exc


class LocalWorld:
    """Several ranks on one GPU in one process (InprocWorld analog, inproc.py:62-127).

    Every segment a rank creates is attached into every other rank's libpgx world,
    so writes are device stores into the peer rank's memory on the same GPU.
    """

    def __init__(self, world_size: int, latency: LatencyModel | None = None, device: int = 0, inline: bool = True,
                 devices=None):
        if world_size < 1:
            raise ConfigError(f"world size must be >= 1, got {world_size}")
        if latency is not None and not latency.is_zero:
            raise ConfigError("latency injection is not supported on the device transport")
        self.world_size = world_size
        self.device_index = device
        self.inline = inline
        # optional rank -> GPU map: several GPUs driven from one process (peer access enabled)
        self.devices = list(devices) if devices is not None else None
        if self.devices is not None:
            if len(self.devices) != world_size:
                raise ConfigError("one device per rank")
            for a in set(self.devices):
                for b in set(self.devices):
                    if a != b:
                        _lib.call("pgx_enable_peer_access", a, b)
        self._transports: dict[int, LocalTransport] = {}
        self._segs: list[tuple[int, Segment]] = []
        self._barrier = threading.Barrier(world_size)
        self._lock = threading.Lock()

    def device_of(self, rank: int) -> int:
        return self.devices[rank] if self.devices is not None else self.device_index

    def transport(self, rank: int) -> LocalTransport:
        if not (0 <= rank < self.world_size):
            raise ConfigError(f"rank {rank} outside world of size {self.world_size}")
        with self._lock:
            if rank in self._transports:
                raise ConfigError(f"transport for rank {rank} already created")
        tr = LocalTransport(self, rank)
        with self._lock:
            self._transports[rank] = tr
            for owner, seg in self._segs:  # segments created before this rank joined
                self._attach(tr, owner, seg)
        return tr

    def _attach(self, tr: LocalTransport, owner: int, seg: Segment) -> None:
        if owner == tr.rank:
            return
        _lib.call("pgx_segment_attach_local", tr.handle, owner, seg.segment_id, seg.data_ptr, seg.flags_ptr,
                  seg.size, seg.notification_count)

    def _publish(self, owner: int, seg: Segment) -> None:
        with self._lock:
            self._segs.append((owner, seg))
            for tr in self._transports.values():
                self._attach(tr, owner, seg)

    def abort_barrier(self) -> None:
        self._barrier.abort()

    def close(self) -> None:
        for tr in list(self._transports.values()):
            tr.close()
        self._transports.clear()


class DistTransport(CudaTransport):
    """One rank per process/GPU; peers are attached through CUDA IPC at the first barrier.

    `group` is a torch.distributed process group used ONLY for the one-time
    handle exchange (plumbing); the data path never touches it.
    """

    def __init__(self, rank: int, world_size: int, device: int, group=None, timeout_s: float = 30.0):
        super().__init__(rank, world_size, device)
        self._group = group
        self._connected = False
        self._timeout = timeout_s
        _lib.call("pgx_world_set_timeout", self.handle, float(timeout_s))

    def connect(self) -> None:
        """Exchange every segment's IPC handle with every peer and attach them."""
        from .rendezvous import exchange

        mine = {}
        shared = getattr(self, "_shared", set())
        for sid in sorted(set(list(self._segments) + [CONTROL_SEGMENT]) - shared):
            buf = (C.c_uint8 * _lib.IPC_HANDLE_BYTES)()
            _lib.call("pgx_segment_export", self.handle, sid, buf)
            d, f, sz, cnt = C.c_void_p(), C.c_void_p(), C.c_uint64(), C.c_uint32()
            _lib.call("pgx_segment_info", self.handle, self.rank, sid, C.byref(d), C.byref(f), C.byref(sz),
                      C.byref(cnt))
            mine[sid] = (bytes(buf), sz.value, cnt.value)
        every = exchange(mine, self.rank, self.world_size, self._group)
        for peer, segs in enumerate(every):
            if peer == self.rank:
                continue
            for sid, (handle, size, count) in segs.items():
                hb = (C.c_uint8 * _lib.IPC_HANDLE_BYTES).from_buffer_copy(handle)
                _lib.call("pgx_segment_attach_ipc", self.handle, peer, sid, hb, size, count)
        self._shared = shared | set(mine)
        self._connected = True

    def sync_segments(self) -> None:
        """Collective: attach the segments every rank created after the first rendezvous
        (e.g. a second exchange object); already-attached ones are not exchanged again."""
        self.connect()

    def _ensure_connected(self, rank: int) -> None:
        if not self._connected and rank != self.rank:
            raise TransportError("peers are not attached yet; call barrier() (rendezvous) first")

    def barrier(self) -> None:
        self.barrier_calls += 1
        if not self._connected:
            self.connect()
        _lib.call("pgx_barrier", self.handle, self.stream.cuda_stream, float(self._timeout))

    def barrier_async(self, stream) -> None:
        """Enqueue the device flag barrier on `stream` without waiting on the host: every
        rank's stream leaves it within one flag round trip (aligns timed regions).  Not
        counted in barrier_calls (measurement only, never on the exchange path)."""
        _lib.call("pgx_barrier_async", self.handle, stream.cuda_stream, float(self._timeout))
