"""Turn-based pipelined data-parallel SGD on the device (reference engine/, pipelined.py).

Same surface as the reference: ``PipelinedRank(config, dataset, transport, recorder)``
with ``begin_iteration(k)``, ``run_turn(layer, gradient)``, ``finalize_iteration()``,
``run() -> RankResult``; ``BarrierRank`` is the phase-separated baseline.  The
protocol (segment layout, notification ids and values, parity double-buffering,
ascending fold gating, consume-once checks, watchdog) follows the reference line
by line in behaviour; every byte it moves and every flop it does runs on the GPU:

* segments are device memory reached through libpgx.so (transport.py);
* sends are one chunked notify-write launch per transfer (pgx_write_notify_chunked);
* folds are ``buffer_axpy`` kernels, the master update is the ``master_update``
  kernel written straight into the model view (no temporaries).

This host-driven engine is the drop-in for the reference's API and protocol
tests.  The throughput path that never polls from the host is
:class:`paper_1706_00095_b200.exchange.DeviceExchange`.
"""

from __future__ import annotations

import time
from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, net
from .config import TrainConfig
from .errors import ConfigError, ProtocolError
from .layout import SEG_GRAD, SEG_MODEL, SEG_WORK, SegmentLayout
from .topology import build_broadcast_tree, build_reduction_tree

_IDLE_SLEEP_S = 2e-5  # runtime.py:27
_TAG_BATCH = 0x6261746368  # engine/sgd.py:24


def batch_indices(seed: int, iteration: int, batch_size: int, dataset_size: int) -> np.ndarray:
    """Global sample indices for one iteration (sgd.py:36-44): splitmix64 stream keyed on
    (seed, TAG_BATCH, iteration), modulo the dataset size, with replacement."""
    m = (1 << 64) - 1
    s = net.derived_seed(seed, _TAG_BATCH, iteration)
    n = np.arange(1, batch_size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(s & m) + n * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (z % np.uint64(dataset_size)).astype(np.int64)


def shard_bounds(batch_size: int, world_size: int, rank: int) -> tuple[int, int]:
    shard = batch_size // world_size
    return rank * shard, (rank + 1) * shard


@dataclass
class RankResult:
    rank: int
    world_size: int
    iterations: int
    model: list
    losses: list
    barrier_calls: int
    fold_counts: list
    wall_ns: int
    events: list = field(default_factory=list)


class TurnState:
    """Communication bookkeeping for one in-flight iteration (runtime.py:45-59)."""

    def __init__(self, num_layers: int, num_children: int):
        self.local_gradient_ready = [False] * num_layers
        self.gradient_forwarded = [False] * num_layers
        self.model_arrived = [False] * num_layers
        self.child_arrived = [set() for _ in range(num_layers)]
        self.next_fold = [0] * num_layers
        self.num_children = num_children
        self.chunks: dict = {}


class RankBase:
    def __init__(self, config: TrainConfig, dataset, transport, recorder=None):
        config.validate()
        if transport.world_size != config.world_size:
            raise ConfigError(f"transport spans {transport.world_size} ranks, config expects {config.world_size}")
        self.cfg = config
        self.dataset = dataset
        self.tr = transport
        self.rec = recorder
        self.rank = transport.rank
        self.specs = config.specs()
        self.num_layers = len(self.specs)
        self.dtype = torch.float64 if config.dtype == "f64" else torch.float32
        self.layout = SegmentLayout([s.param_count for s in self.specs], config.chunk_bytes, config.elem_bytes)
        red = build_reduction_tree(config.world_size)
        bc = build_broadcast_tree(config.world_size)
        self.red_children = red.children[self.rank]
        self.red_parent = red.parent.get(self.rank)
        self.bc_children = bc.children[self.rank]
        self.bc_parent = bc.parent.get(self.rank)
        self.is_master = self.rank == 0
        self.parent_slot = None if self.red_parent is None else red.children[self.red_parent].index(self.rank)
        self.parent_child_count = 0 if self.red_parent is None else len(red.children[self.red_parent])

        lay = self.layout
        nc = len(self.red_children)
        self.seg_work = transport.segment_create(SEG_WORK, lay.work_size, 1)
        self.seg_model = transport.segment_create(SEG_MODEL, lay.model_rx_size, lay.model_notif_count)
        self.seg_grad = transport.segment_create(SEG_GRAD, lay.grad_rx_size(nc), lay.grad_notif_count(nc))
        eb = lay.elem_bytes
        self.model_views = [self.seg_work.view(self.dtype, lay.work_model_offset(l), self.specs[l].param_count)
                            for l in range(self.num_layers)]
        self.grad_views = [self.seg_work.view(self.dtype, lay.work_grad_offset(l), self.specs[l].param_count)
                           for l in range(self.num_layers)]
        self.model_region = self.seg_work.view(self.dtype, 0, lay.total_params)
        self.grad_region = self.seg_work.view(self.dtype, lay.total_bytes, lay.total_params)
        assert lay.total_bytes == lay.total_params * eb
        with self._stream():
            start = net.init_model(config.seed, self.specs, self.dtype, self.tr.device)
            for l in range(self.num_layers):
                self.model_views[l].copy_(start[l])
        self.tr.stream.synchronize()
        self._grad_poll_span = (1, lay.grad_notif_count(nc) - 1)
        self._model_poll_span = (1, lay.model_notif_count - 1)
        self.losses: list = []
        self.fold_counts = [0] * self.num_layers
        self._tickets: list = []
        self._flights: list = []
        self.k = 0
        self.parity = 0

    @contextmanager
    def _stream(self):
        with torch.cuda.device(self.tr.device), torch.cuda.stream(self.tr.stream):
            yield

    # -- receive-slot views (runtime.py:161-177) --------------------------------
    def _grad_rx(self, slot: int, layer: int, parity: int) -> torch.Tensor:
        return self.seg_grad.view(self.dtype, self.layout.grad_slot_offset(slot, layer, parity),
                                  self.specs[layer].param_count)

    def _grad_bulk_rx(self, slot: int, parity: int) -> torch.Tensor:
        return self.seg_grad.view(self.dtype, self.layout.grad_bulk_offset(slot, parity), self.layout.total_params)

    def _model_rx(self, layer: int, parity: int) -> torch.Tensor:
        return self.seg_model.view(self.dtype, self.layout.model_slot_offset(layer, parity),
                                   self.specs[layer].param_count)

    def _model_bulk_rx(self, parity: int) -> torch.Tensor:
        return self.seg_model.view(self.dtype, self.layout.model_bulk_offset(parity), self.layout.total_params)

    def _record(self, kind: str, layer: int, t0: int, t1: int) -> None:
        if self.rec is not None:
            self.rec.record(kind, self.k, layer, t0, t1)

    # -- device arithmetic --------------------------------------------------------
    def _axpy(self, x: torch.Tensor, y: torch.Tensor) -> None:
        fn = "pgx_axpy_f64" if self.dtype == torch.float64 else "pgx_axpy_f32"
        _lib.call(fn, 1.0, x.data_ptr(), y.data_ptr(), y.numel(), self.tr.stream.cuda_stream)

    def _update(self, w: torch.Tensor, g: torch.Tensor) -> None:
        fn = "pgx_master_update_f64" if self.dtype == torch.float64 else "pgx_master_update_f32"
        _lib.call(fn, w.data_ptr(), g.data_ptr(), float(self.cfg.epsilon), w.data_ptr(), w.numel(),
                  self.tr.stream.cuda_stream)

    # -- sending (runtime.py:185-278) --------------------------------------------------
    def _send(self, dest_rank, remote_segment, remote_offset, local_offset, nbytes, notif_base, kind, layer):
        t0 = time.monotonic_ns()
        ticket = self.tr.write_notify_chunked(SEG_WORK, local_offset, dest_rank, remote_segment, remote_offset,
                                              nbytes, self.layout.chunk_bytes, notif_base, self.k + 1)
        self._tickets.append(ticket)
        self._flights.append((kind, self.k, layer, t0, [ticket]))

    def _send_gradient_layer(self, layer: int) -> None:
        lay = self.layout
        self._send(self.red_parent, SEG_GRAD, lay.grad_slot_offset(self.parent_slot, layer, self.parity),
                   lay.work_grad_offset(layer), lay.layer_bytes[layer],
                   lay.grad_notif_base(self.parent_slot, layer, self.parity), "send_trigger", layer)

    def _send_model_layer(self, layer: int) -> None:
        lay = self.layout
        for child in self.bc_children:
            self._send(child, SEG_MODEL, lay.model_slot_offset(layer, self.parity), lay.work_model_offset(layer),
                       lay.layer_bytes[layer], lay.model_notif_base(layer, self.parity), "model_forward", layer)

    def _send_gradient_bulk(self) -> None:
        lay = self.layout
        self._send(self.red_parent, SEG_GRAD, lay.grad_bulk_offset(self.parent_slot, self.parity), lay.total_bytes,
                   lay.total_bytes, lay.grad_bulk_base(self.parent_child_count, self.parent_slot, self.parity),
                   "send_trigger", -1)

    def _send_model_bulk(self) -> None:
        lay = self.layout
        for child in self.bc_children:
            self._send(child, SEG_MODEL, lay.model_bulk_offset(self.parity), 0, lay.total_bytes,
                       lay.model_bulk_base(self.parity), "model_forward", -1)

    def _wait_tickets(self) -> None:
        if self._tickets:
            self.tr.ticket_wait_all(self._tickets, timeout=self.cfg.finalize_timeout_s)
        if self.rec is not None:
            for kind, k, layer, t0, tickets in self._flights:
                t1 = max(t.completed_at_ns for t in tickets)
                self.rec.record(kind, k, layer, t0, max(t0, t1))
        self._tickets = []
        self._flights = []

    # -- batches -----------------------------------------------------------------
    def _shard(self, k: int):
        idx = batch_indices(self.cfg.seed, k, self.cfg.batch_size, len(self.dataset))
        lo, hi = shard_bounds(self.cfg.batch_size, self.cfg.world_size, self.rank)
        return self.dataset.take(idx[lo:hi])

    def _inflate(self) -> None:
        if self.cfg.compute_inflation_ns > 0:
            time.sleep(self.cfg.compute_inflation_ns * 1e-9)

    def _train_iteration(self, k: int) -> None:
        raise NotImplementedError

    def run(self) -> RankResult:
        """Rendezvous barrier (not counted), then the loop (runtime.py:311-335)."""
        if self.cfg.world_size > 1:
            self.tr.barrier()
        base_barriers = self.tr.barrier_calls
        t0 = time.monotonic_ns()
        for k in range(self.cfg.iterations):
            self._train_iteration(k)
        self.tr.stream.synchronize()
        wall_ns = time.monotonic_ns() - t0
        return RankResult(
            rank=self.rank, world_size=self.cfg.world_size, iterations=self.cfg.iterations,
            model=[v.detach().cpu().numpy().copy() for v in self.model_views],
            losses=list(self.losses), barrier_calls=self.tr.barrier_calls - base_barriers,
            fold_counts=list(self.fold_counts), wall_ns=wall_ns,
            events=list(self.rec.events) if self.rec is not None else [])

    # -- notification consumption (runtime.py:339-363) -------------------------------
    def _consume(self, segment_id: int, span):
        hits = self.tr.notify_poll(segment_id, span[0], span[1])
        out = []
        nc = len(self.red_children)
        for nid, value in hits:
            desc = (self.layout.decode_grad_id(nid, nc) if segment_id == SEG_GRAD
                    else self.layout.decode_model_id(nid))
            if desc is None:
                raise ProtocolError(f"rank {self.rank}: unassigned notification id {nid}")
            parity = desc[3]
            if value == self.k + 2 and parity == (self.k + 1) & 1:
                continue  # next iteration's data, left pending
            if value != self.k + 1 or parity != self.parity:
                raise ProtocolError(f"rank {self.rank}: iteration {self.k} saw notification value "
                                    f"{value} on id {nid} (parity {parity})")
            self.tr.notify_reset(segment_id, nid)
            out.append(desc)
        return out


class PipelinedRank(RankBase):
    """Layer-wise pipelined schedule (pipelined.py:43-218)."""

    def begin_iteration(self, k: int) -> None:
        self.k = k
        self.parity = k & 1
        self.state = TurnState(self.num_layers, len(self.red_children))

    def run_turn(self, layer: int, gradient) -> None:
        """Publish one layer's local gradient and advance communication (pipelined.py:49-58)."""
        with self._stream():
            g = torch.as_tensor(gradient, device=self.tr.device, dtype=self.dtype)
            self.grad_views[layer].copy_(g.reshape(-1))
        self.state.local_gradient_ready[layer] = True
        if self.cfg.world_size == 1:
            self._apply_update(layer)
            self.state.gradient_forwarded[layer] = True
            self.state.model_arrived[layer] = True
            return
        self._comm_pass()

    def finalize_iteration(self) -> None:
        """Poll until the iteration's obligations are met; watchdog (pipelined.py:60-80)."""
        t0 = time.monotonic_ns()
        deadline = time.monotonic() + self.cfg.finalize_timeout_s
        while not self._iteration_done():
            if self._comm_pass():
                deadline = time.monotonic() + self.cfg.finalize_timeout_s
            elif time.monotonic() > deadline:
                raise ProtocolError(f"rank {self.rank}: no progress for {self.cfg.finalize_timeout_s:.1f}s "
                                    f"finishing iteration {self.k}: {self._dump_state()}")
            else:
                time.sleep(_IDLE_SLEEP_S)
        self._wait_tickets()
        self._record("finalize", -1, t0, time.monotonic_ns())

    def _train_iteration(self, k: int) -> None:
        self.begin_iteration(k)
        x, t = self._shard(k)
        t0 = time.monotonic_ns()
        with self._stream():
            _, cache = net.forward(self.specs, self.model_views, x)
        self._record("forward", -1, t0, time.monotonic_ns())
        self._turn_clock = time.monotonic_ns()

        def emit(layer, gradient):
            self._inflate()
            self._record("backward_layer", layer, self._turn_clock, time.monotonic_ns())
            self.run_turn(layer, gradient)
            self._turn_clock = time.monotonic_ns()

        with self._stream():
            _, loss = net.backward_from_cache(self.specs, self.model_views, cache, t, emit)
        self.losses.append(float(loss))
        self.finalize_iteration()

    def _apply_update(self, layer: int) -> None:
        t0 = time.monotonic_ns()
        with self._stream():
            self._update(self.model_views[layer], self.grad_views[layer])
        self._record("master_update", layer, t0, time.monotonic_ns())

    def _comm_pass(self) -> bool:
        t_pass = time.monotonic_ns()
        st = self.state
        progressed = False
        if self.red_children:
            for kind, slot, layer, _p in self._consume(SEG_GRAD, self._grad_poll_span):
                if kind != "layer":
                    raise ProtocolError(f"rank {self.rank}: whole-model gradient chunk during a layer-wise run")
                progressed = True
                if self._count_chunk(("g", slot, layer), self.layout.layer_chunks[layer]):
                    st.child_arrived[layer].add(slot)
                    self._record("recv_notify", layer, t_pass, time.monotonic_ns())
        arrived = []
        if self.bc_parent is not None:
            for kind, _s, layer, _p in self._consume(SEG_MODEL, self._model_poll_span):
                if kind != "layer":
                    raise ProtocolError(f"rank {self.rank}: whole-model broadcast chunk during a layer-wise run")
                progressed = True
                if self._count_chunk(("m", layer), self.layout.layer_chunks[layer]):
                    arrived.append(layer)
        self._advance_folds()
        for layer in sorted(arrived):
            self._handle_model_arrival(layer, t_pass)
        return progressed

    def _count_chunk(self, key, target: int) -> bool:
        seen = self.state.chunks.get(key, 0) + 1
        if seen > target:
            raise ProtocolError(f"rank {self.rank}: transfer {key} delivered more than its {target} chunks")
        self.state.chunks[key] = seen
        return seen == target

    def _advance_folds(self) -> None:
        """Ascending, gated folds (pipelined.py:158-177)."""
        st = self.state
        for layer in range(self.num_layers):
            if not st.local_gradient_ready[layer] or st.gradient_forwarded[layer]:
                continue
            while st.next_fold[layer] < st.num_children and st.next_fold[layer] in st.child_arrived[layer]:
                slot = st.next_fold[layer]
                t0 = time.monotonic_ns()
                with self._stream():
                    self._axpy(self._grad_rx(slot, layer, self.parity), self.grad_views[layer])
                self._record("reduce_local", layer, t0, time.monotonic_ns())
                self.fold_counts[layer] += 1
                st.next_fold[layer] += 1
            if st.next_fold[layer] == st.num_children:
                self._complete_gradient(layer)

    def _complete_gradient(self, layer: int) -> None:
        st = self.state
        if self.is_master:
            self._apply_update(layer)
            if self.bc_children:
                self._send_model_layer(layer)
            st.model_arrived[layer] = True
        else:
            self._send_gradient_layer(layer)
        st.gradient_forwarded[layer] = True

    def _handle_model_arrival(self, layer: int, t_pass: int) -> None:
        st = self.state
        if st.model_arrived[layer]:
            raise ProtocolError(f"rank {self.rank}: duplicate model update for layer {layer}")
        if not st.gradient_forwarded[layer]:
            raise ProtocolError(f"rank {self.rank}: model layer {layer} arrived before this rank's "
                                "gradient contribution went up")
        self._record("recv_notify", layer, t_pass, time.monotonic_ns())
        with self._stream():
            self.model_views[layer].copy_(self._model_rx(layer, self.parity))
        if self.bc_children:
            self._send_model_layer(layer)
        st.model_arrived[layer] = True

    def _iteration_done(self) -> bool:
        st = self.state
        return all(st.gradient_forwarded) and all(st.model_arrived)

    def _dump_state(self) -> str:
        st = self.state
        waiting = []
        for layer in range(self.num_layers):
            if not st.gradient_forwarded[layer]:
                missing = [c for c in range(st.num_children) if c not in st.child_arrived[layer]]
                waiting.append(f"layer {layer} gradient (children pending: {missing})")
            elif not st.model_arrived[layer]:
                waiting.append(f"layer {layer} model update")
        return "; ".join(waiting) or "nothing pending"


class BarrierRank(RankBase):
    """Phase-separated baseline: backward, barrier, bulk reduce/update/broadcast, barrier
    (engine/barrier.py:24-141)."""

    def _train_iteration(self, k: int) -> None:
        self.k = k
        self.parity = k & 1
        self._bulk_counts: dict = {}
        x, t = self._shard(k)
        t0 = time.monotonic_ns()
        with self._stream():
            _, cache = net.forward(self.specs, self.model_views, x)
        self._record("forward", -1, t0, time.monotonic_ns())
        self._turn_clock = time.monotonic_ns()

        def emit(layer, gradient):
            self._inflate()
            self._record("backward_layer", layer, self._turn_clock, time.monotonic_ns())
            self.grad_views[layer].copy_(gradient.reshape(-1))
            self._turn_clock = time.monotonic_ns()

        with self._stream():
            _, loss = net.backward_from_cache(self.specs, self.model_views, cache, t, emit)
        self.losses.append(float(loss))
        self._fence()
        if self.cfg.world_size == 1:
            for layer in range(self.num_layers):
                self._apply_update(layer)
        else:
            self._exchange()
            self._wait_tickets()
        self._fence()

    def _fence(self) -> None:
        t0 = time.monotonic_ns()
        self.tr.barrier()
        self._record("barrier", -1, t0, time.monotonic_ns())

    def _apply_update(self, layer: int) -> None:
        t0 = time.monotonic_ns()
        with self._stream():
            self._update(self.model_views[layer], self.grad_views[layer])
        self._record("master_update", layer, t0, time.monotonic_ns())

    def _exchange(self) -> None:
        for slot in range(len(self.red_children)):
            self._wait_bulk(("gb", slot))
            t0 = time.monotonic_ns()
            with self._stream():
                self._axpy(self._grad_bulk_rx(slot, self.parity), self.grad_region)
            self._record("reduce_local", -1, t0, time.monotonic_ns())
            for layer in range(self.num_layers):
                self.fold_counts[layer] += 1
        if self.is_master:
            for layer in range(self.num_layers):
                self._apply_update(layer)
            if self.bc_children:
                self._send_model_bulk()
        else:
            self._send_gradient_bulk()
            self._wait_bulk(("mb",))
            with self._stream():
                self.model_region.copy_(self._model_bulk_rx(self.parity))
            if self.bc_children:
                self._send_model_bulk()

    def _wait_bulk(self, key) -> None:
        target = self.layout.bulk_chunks
        t0 = time.monotonic_ns()
        deadline = time.monotonic() + self.cfg.finalize_timeout_s
        while self._bulk_counts.get(key, 0) < target:
            if self._pump():
                deadline = time.monotonic() + self.cfg.finalize_timeout_s
            elif time.monotonic() > deadline:
                raise ProtocolError(f"rank {self.rank}: no progress for {self.cfg.finalize_timeout_s:.1f}s "
                                    f"waiting on transfer {key} in iteration {self.k}")
            else:
                time.sleep(_IDLE_SLEEP_S)
        self._record("recv_notify", -1, t0, time.monotonic_ns())

    def _pump(self) -> bool:
        progressed = False
        if self.red_children:
            for kind, slot, _l, _p in self._consume(SEG_GRAD, self._grad_poll_span):
                if kind != "bulk":
                    raise ProtocolError(f"rank {self.rank}: layer-wise gradient chunk during a whole-model run")
                self._count_bulk(("gb", slot))
                progressed = True
        if self.bc_parent is not None:
            for kind, _s, _l, _p in self._consume(SEG_MODEL, self._model_poll_span):
                if kind != "bulk":
                    raise ProtocolError(f"rank {self.rank}: layer-wise broadcast chunk during a whole-model run")
                self._count_bulk(("mb",))
                progressed = True
        return progressed

    def _count_bulk(self, key) -> None:
        seen = self._bulk_counts.get(key, 0) + 1
        if seen > self.layout.bulk_chunks:
            raise ProtocolError(f"rank {self.rank}: transfer {key} delivered more than its "
                                f"{self.layout.bulk_chunks} chunks")
        self._bulk_counts[key] = seen
