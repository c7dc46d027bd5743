"""DeviceExchange — the device-driven per-layer exchange, wired into PyTorch.

This is the throughput path of the package: the
reference's per-layer turn (pipelined.py:49-58 publish, :158-188 fold/update,
:190-203 model arrival) becomes one kernel launch per layer on a high-priority
communication stream, issued from a post-accumulate-grad hook the moment the
layer's gradient is final (the `on_layer` contract, net.py:163-172), with all
waiting done on the device.  The reference's barrier-free `finalize_iteration`
drain (pipelined.py:60-80) becomes a per-layer *gate* in the next iteration's
forward-pre-hook: layer l's forward waits only for layer l's new weights.

Weights live in the library's IPC-exported flat model buffer ([W row-major][b]
per layer, the reference layout net.py:57-63) so peers install updated shards
directly into them; gradients are read where autograd left them.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import ConfigError, ShapeError

VARIANTS = {"tree": _lib.VARIANT_TREE, "twoshot": _lib.VARIANT_TWOSHOT, "twoshot_ce": _lib.VARIANT_TWOSHOT_CE,
            "nvls": _lib.VARIANT_NVLS, "oneshot": _lib.VARIANT_ONESHOT, "twoshot_cep": _lib.VARIANT_TWOSHOT_CEP,
            "oneshot_ll": _lib.VARIANT_ONESHOT_LL, "oneshot_l128": _lib.VARIANT_ONESHOT_L128,
            "twoshot_bulk": _lib.VARIANT_TWOSHOT_BULK, "twoshot_l128": _lib.VARIANT_TWOSHOT_L128,
            # TWOSHOT_BULK with its reduce-scatter on the copy engines (the bulk_ce_rs flag)
            "twoshot_ceb": _lib.VARIANT_TWOSHOT_BULK,
            # TWOSHOT_CE with the owner fold fed by TMA loads on a capped grid (the ce_tma_owner flag)
            "twoshot_cet": _lib.VARIANT_TWOSHOT_CE}
VARIANT_ALIASES = {"twoshot_ceb": ("twoshot_bulk", "bulk_ce_rs"),  # Python name -> (library variant, flag)
                   "twoshot_cet": ("twoshot_ce", "ce_tma_owner")}
FLAGS = {"ce_rs_parts": _lib.XF_CE_RS_PARTS, "tma": _lib.XF_TMA, "oneshot_small_chunks": _lib.XF_ONESHOT_SMALL_CHUNKS,
         "auto_chunk_tree": _lib.XF_AUTO_CHUNK_TREE, "no_auto_chunk_nvls": _lib.XF_NO_AUTO_CHUNK_NVLS,
         "allow_l128": _lib.XF_ALLOW_L128, "bulk_lean": _lib.XF_BULK_LEAN, "bulk_ce_rs": _lib.XF_BULK_CE_RS,
         "ce_tma_owner": _lib.XF_CE_TMA_OWNER, "lean_capped": _lib.XF_LEAN_CAPPED}
MODES = {"ref64": _lib.MODE_REF64, "ref32": _lib.MODE_REF32, "fast32": _lib.MODE_FAST32, "sum32": _lib.MODE_SUM32}


# Layers of (64 K, 1 M) elements take the 128-byte-line two-shot when the caller opts in
# (allow_l128): 1-16 MB device time below NCCL's all-reduce at N=2 and N=4
# (profiles/r5s_sweep_mid_n*.jsonl); slower than the SM two-shot at 64 MB+ (r5u_sweep_large).
L128_BAND = ((1 << 16) + 1, 1 << 20)


def choose_variant(elems: int, world: int, tree_below: int = 0, ce_from: int = 1 << 20,
                   oneshot_below: int | None = None, large: str = "ce", ll_below: int = 0,
                   l128_range: tuple[int, int] = (0, 0)) -> str:
    """Layer-size policy (measured, profiles/r1*_sweep*): the smallest layers are pure
    latency and take the one-shot exchange (one NVLink hop); mid-size layers the SM
    two-shot kernel; layers of `ce_from` elements or more move their shards with the copy
    engines, which do not take SMs away from the backward kernels they overlap with.
    `tree_below` optionally keeps the paper's tree for the smallest layers.  `ll_below`
    (fp32 modes; DeviceExchange passes 64 K elements) sends the smallest layers as LL words
    (profiles/r3v: 14–21 µs up to 256 KB at N=4, NCCL 17–23).  large="sm"
    keeps the SM two-shot for the large layers too (run with a CTA cap and big chunks,
    see DeviceExchange `large_ctas`); large="cep" moves the reduce-scatter by copy engine
    and runs fold + update + all-gather as the SM owner kernel on a capped grid;
    large="bulk" moves every byte with TMA bulk copies from a capped grid (TWOSHOT_BULK);
    large="ceb" is TWOSHOT_BULK with the reduce-scatter on the copy engines (DeviceExchange
    adds the bulk_ce_rs flag): the kernel only folds, updates and all-gathers.
    `l128_range` = [lo, hi) elements sent by the fence-free 128-byte-line two-shot
    (TWOSHOT_L128; DeviceExchange passes it only with the allow_l128 flag)."""
    if oneshot_below is None:  # one-shot moves (N-1)*S per GPU: the crossover shrinks with N
        oneshot_below = (1 << 20) // max(world, 1)  # N=4: 1 MB layers (profiles/r2b_sweep_n4)
    if world > 1 and elems < tree_below:
        return "tree"
    if world > 1 and elems <= ll_below:  # fence-free LL words: lowest latency up to ~256 KB
        return "oneshot_ll"
    if world > 1 and l128_range[0] <= elems < l128_range[1]:
        return "twoshot_l128"
    if world > 1 and elems < oneshot_below:
        return "oneshot"
    if world > 1 and elems >= ce_from:
        return {"ce": "twoshot_ce", "cep": "twoshot_cep", "sm": "twoshot", "bulk": "twoshot_bulk",
                "ceb": "twoshot_ceb", "cet": "twoshot_cet"}[large]
    return "twoshot"


def layer_ctas(elems, world: int, *, large_from: int = 1 << 20, large_ctas: int = 0, overlap_ctas: int = 0,
               overlap_exposed: int = 1) -> list[int]:
    """Per-layer CTA caps (0 = the library default) of an exchange plan: layers of
    >= `large_from` elements get `large_ctas`; with `overlap_ctas` (N > 1) every smaller layer
    but the first `overlap_exposed` ones (the last gradients backward emits, whose exchange
    nothing hides) runs on at most `overlap_ctas` CTAs (DeviceExchange, variant="auto")."""
    caps = []
    for l, n in enumerate(elems):
        if n >= large_from:
            caps.append(int(large_ctas))
        elif overlap_ctas > 0 and world > 1 and l >= max(1, overlap_exposed):
            caps.append(int(overlap_ctas))
        else:
            caps.append(0)
    return caps


class DeviceExchange:
    def __init__(self, transport, layer_elems, *, mode: str = "fast32", variant="twoshot",
                 chunk_elems: int = 16384, lr: float = 0.01, scale: float | None = None,
                 momentum: float = 0.0, weight_decay: float = 0.0, seg_base: int = 16, max_ctas: int = 0,
                 tree_below: int = 0, low_priority_from: int | None = None, large: str = "ce",
                 large_from: int = 1 << 20, large_ctas: int = 0, large_chunk_elems: int = 0,
                 layer_chunk_elems=None, layer_max_ctas=None, ce_parts: int = 0, ce_rs_streams: int = 0,
                 flags=(), l128_range: tuple[int, int] = (0, 0), overlap_ctas: int = 16,
                 overlap_exposed: int = 1):
        """variant: one name, a per-layer list, or "auto" (choose_variant; `large` = "ce" or
        "sm" for layers of >= `large_from` elements).  Layers of >= `large_from` elements get
        `large_chunk_elems` / `large_ctas` (0 = the global chunk_elems / max_ctas): fewer CTAs
        with bigger chunks move the same bytes with far fewer per-chunk system fences
        (profiles/r3e), leaving SMs to the backward kernels.  layer_chunk_elems /
        layer_max_ctas override per layer (0 = default).  ce_parts / ce_rs_streams / flags
        (names of FLAGS) are the library's tuning knobs (pgx_xchg_config, ABI 3); the
        defaults are the measured choices.  `overlap_ctas` (variant="auto", N > 1): CTA cap of
        the small layers (< `large_from`) whose exchange overlaps the rest of the backward —
        every layer but layer 0, the last one backward emits, whose exchange nothing hides and
        which keeps the full grid.  Fewer CTAs per hidden exchange leave the SMs to the
        backward kernels (GoogLeNet N=4: 16 CTAs 9.67 ms/step vs 9.82-9.87 uncapped, AlexNet
        N=4: 5.00-5.02 vs 5.05-5.07 ms, r6j/r6k); 0 = every layer on the full grid.
        `overlap_exposed`: how many of the first layers (the last ones backward emits) keep
        the full grid."""
        if mode not in MODES:
            raise ConfigError(f"mode must be one of {sorted(MODES)}, got {mode!r}")
        flags = tuple(flags)
        self.tr = transport
        self.world = transport.world_size
        self.rank = transport.rank
        self.mode = mode
        self.layer_elems = [int(n) for n in layer_elems]
        L = len(self.layer_elems)
        auto = isinstance(variant, str) and variant == "auto"
        if auto:
            ll = (1 << 16) if mode != "ref64" else 0
            l128 = tuple(l128_range) if ("allow_l128" in flags and mode != "ref64") else (0, 0)
            variants = [choose_variant(n, self.world, tree_below, ce_from=large_from, large=large, ll_below=ll,
                                       l128_range=l128) for n in self.layer_elems]
        elif isinstance(variant, str):
            variants = [variant] * L
        else:
            variants = list(variant)
        if len(variants) != L or any(v not in VARIANTS for v in variants):
            raise ConfigError(f"bad variant list {variants}")
        if "twoshot_ceb" in variants:  # one library flag switches every bulk layer's reduce-scatter
            if "twoshot_bulk" in variants:
                raise ConfigError("twoshot_bulk and twoshot_ceb layers cannot be mixed in one exchange")
            if "bulk_ce_rs" not in flags:
                flags += ("bulk_ce_rs",)
        if "twoshot_cet" in variants:  # one library flag switches every copy-engine layer's owner fold
            if "twoshot_ce" in variants:
                raise ConfigError("twoshot_ce and twoshot_cet layers cannot be mixed in one exchange")
            if "ce_tma_owner" not in flags:
                flags += ("ce_tma_owner",)
        self.variants = variants
        self.scale = 1.0 / self.world if scale is None else float(scale)
        self._elems = (C.c_uint64 * L)(*self.layer_elems)
        self._vars = (C.c_int * L)(*[VARIANTS[v] for v in variants])
        big = [n >= large_from for n in self.layer_elems]
        chunks = list(layer_chunk_elems) if layer_chunk_elems is not None else \
            [int(large_chunk_elems) if b else 0 for b in big]
        ctas = list(layer_max_ctas) if layer_max_ctas is not None else \
            layer_ctas(self.layer_elems, self.world, large_from=large_from, large_ctas=large_ctas,
                       overlap_ctas=overlap_ctas if (auto and not max_ctas) else 0, overlap_exposed=overlap_exposed)
        if len(chunks) != L or len(ctas) != L:
            raise ConfigError("layer_chunk_elems / layer_max_ctas need one entry per layer")
        self._chunks_req = [int(c) for c in chunks]
        self.layer_max_ctas = [int(c) or int(max_ctas) for c in ctas]
        self._chunks = (C.c_uint64 * L)(*[int(c) for c in chunks])
        self._ctas = (C.c_int * L)(*[int(c) for c in ctas])
        cfg = _lib.XchgConfig(
            num_layers=L, layer_elems=self._elems, variant=self._vars, mode=MODES[mode],
            chunk_elems=int(chunk_elems), lr=float(lr), scale=self.scale, momentum=float(momentum),
            weight_decay=float(weight_decay), seg_base=int(seg_base), max_ctas=int(max_ctas),
            layer_chunk_elems=self._chunks, layer_max_ctas=self._ctas, ce_parts=int(ce_parts),
            ce_rs_streams=int(ce_rs_streams), flags=self._flag_bits(flags))
        h = C.c_void_p()
        _lib.call("pgx_xchg_create", transport.handle, C.byref(cfg), C.byref(h))
        self.handle = h
        self.seg_ids = (seg_base, seg_base + 1)
        for sid in self.seg_ids:
            transport.adopt_segment(sid)
        mp = C.c_void_p()
        offs = (C.c_uint64 * L)()
        _lib.call("pgx_xchg_model", h, C.byref(mp), offs)
        self.model_offsets = [int(o) for o in offs]
        self.dtype = torch.float64 if mode == "ref64" else torch.float32
        seg = transport.segment(seg_base)
        eb = torch.empty((), dtype=self.dtype).element_size()
        self.model = seg.data[: (seg.size // eb) * eb].view(self.dtype)
        if "nvls" in variants:
            self._nvls_setup()  # the weights move into the multicast-backed buffer
            _lib.call("pgx_xchg_model", h, C.byref(mp), offs)
            from .transport import _CudaArray
            self._nvls_model = torch.as_tensor(_CudaArray(mp.value, seg.size, self), device=transport.device)
            self.model = self._nvls_model[: (seg.size // eb) * eb].view(self.dtype)
        self.layer_views = [self.model[o:o + n] for o, n in zip(self.model_offsets, self.layer_elems)]
        with torch.cuda.device(transport.device):
            self.stream = torch.cuda.Stream(device=transport.device, priority=-1)
            # optional: large layers (long slack before their next use) launch at normal priority
            # so their CTAs fill gaps instead of pre-empting the backward kernels
            self.stream_low = torch.cuda.Stream(device=transport.device, priority=0)
        self.low_priority_from = low_priority_from
        self._capture_keep: list = []  # gradient pieces read by captured launches
        self.connected = False
        self.device_iteration = False
        self.launches = 0
        # The library's side streams (tree down pass, copy-engine push, owner side) are torch
        # streams, so the caching allocator can track gradient pieces used on them.
        with torch.cuda.device(transport.device):
            self.internal_streams = [torch.cuda.Stream(device=transport.device, priority=-1)
                                     for _ in range(_lib.XCHG_STREAMS)]
        arr = (C.c_void_p * _lib.XCHG_STREAMS)(*[s.cuda_stream for s in self.internal_streams])
        _lib.call("pgx_xchg_set_streams", h, arr, _lib.XCHG_STREAMS)

    @staticmethod
    def _flag_bits(flags) -> int:
        bits = 0
        for f in flags:
            if f not in FLAGS:
                raise ConfigError(f"unknown exchange flag {f!r}; known: {sorted(FLAGS)}")
            bits |= FLAGS[f]
        return bits

    def ce_parts(self, layer: int) -> int:
        """Pipelined owner parts of this rank's shard (copy-engine layers; 1 otherwise)."""
        n = C.c_int()
        _lib.call("pgx_xchg_layer_parts", self.handle, layer, C.byref(n))
        return n.value

    def _nvls_setup(self) -> None:
        """Collective: rank 0's multicast handle reaches every rank as a file descriptor over
        a Unix socket (SCM_RIGHTS); every rank adds its GPU; after all did, bind memory."""
        import os
        import socket

        import torch.distributed as dist

        if self.world < 2 or not dist.is_initialized():
            raise ConfigError("the NVLS variant needs >= 2 ranks in an initialised torch.distributed group")
        fd = C.c_int(-1)
        _lib.call("pgx_xchg_nvls_export", self.handle, C.byref(fd))
        token = [f"pgx-nvls-{os.getpid()}-{id(self)}" if self.rank == 0 else None]
        dist.broadcast_object_list(token, src=0)
        addr = "\0" + token[0]
        if self.rank == 0:
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(addr)
            srv.listen(self.world)
            dist.barrier()
            for _ in range(self.world - 1):
                conn, _ = srv.accept()
                socket.send_fds(conn, [b"x"], [fd.value])
                conn.close()
            srv.close()
            os.close(fd.value)
            got = -1
        else:
            dist.barrier()
            cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            cli.connect(addr)
            _, fds, _, _ = socket.recv_fds(cli, 1, 1)
            cli.close()
            got = fds[0]
        _lib.call("pgx_xchg_nvls_import", self.handle, got)
        dist.barrier()  # every GPU joined the multicast team before anyone binds
        _lib.call("pgx_xchg_nvls_bind", self.handle)
        dist.barrier()

    # -- wiring ----------------------------------------------------------------
    def connect(self) -> None:
        """After the transport's rendezvous: resolve every rank's segments."""
        _lib.call("pgx_xchg_connect", self.handle)
        self.connected = True

    def layer_bytes(self, layer: int) -> tuple[int, int]:
        nvl, hbm = C.c_uint64(), C.c_uint64()
        _lib.call("pgx_xchg_layer_bytes", self.handle, layer, C.byref(nvl), C.byref(hbm))
        return nvl.value, hbm.value

    def layer_plan(self, layer: int) -> tuple[int, int]:
        """(effective chunk elements, CTAs of the layer's kernel launch)."""
        ch, ctas = C.c_uint64(), C.c_int()
        _lib.call("pgx_xchg_layer_plan", self.handle, layer, C.byref(ch), C.byref(ctas))
        return ch.value, ctas.value

    # -- per-layer operations ------------------------------------------------------
    def stream_for(self, layer: int):
        """The launch stream of a layer (high priority unless it is a large, slack-rich layer)."""
        if self.low_priority_from is not None and self.layer_elems[layer] >= self.low_priority_from:
            return self.stream_low
        return self.stream

    def launch(self, layer: int, iteration: int, pieces, stream=None, phases: int = _lib.PHASE_ALL) -> None:
        """Exchange layer `layer` of iteration `iteration`; `pieces` are device tensors
        covering the layer's flat gradient in order (e.g. [dW, db])."""
        n = len(pieces)
        if not 1 <= n <= _lib.MAX_PIECES:
            raise ShapeError(f"1..{_lib.MAX_PIECES} gradient pieces, got {n}")
        for p in pieces:
            if p.dtype != self.dtype or not p.is_cuda:
                raise ShapeError(f"gradient pieces must be {self.dtype} CUDA tensors")
            if not p.is_contiguous():
                raise ShapeError("gradient pieces must be contiguous")
        ptrs = (C.c_void_p * n)(*[p.data_ptr() for p in pieces])
        cnts = (C.c_uint64 * n)(*[p.numel() for p in pieces])
        st = stream or self.stream_for(layer)
        _lib.call("pgx_xchg_layer", self.handle, layer, iteration & 0xFFFFFFFF, ptrs, cnts, n, phases, st.cuda_stream)
        if not torch.cuda.is_current_stream_capturing():
            # the pieces are read asynchronously on the launch stream and, for the copy-engine
            # variant, on internal streams: keep the caching allocator from recycling them early
            for p in pieces:
                p.record_stream(st)
                for s in self.internal_streams:
                    p.record_stream(s)
        else:
            # inside a capture record_stream does not order frees: a piece freed now would be
            # handed to a later allocation of the same graph while the replayed exchange still
            # reads it, so captured pieces live as long as this exchange (the graph's memory)
            self._capture_keep.extend(pieces)
        self.launches += 1

    def set_device_iteration(self, enable: bool, current: int) -> None:
        """Graph mode: epochs come from a device counter (`current` = last launched
        iteration); capture `tick()` at the start of every step."""
        _lib.call("pgx_xchg_device_iteration", self.handle, int(bool(enable)), current & 0xFFFFFFFF)
        self.device_iteration = bool(enable)

    def tick(self, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.tr.device)
        _lib.call("pgx_xchg_tick", self.handle, s.cuda_stream)

    def gate_all(self, iteration: int, stream=None) -> None:
        """One launch gating `stream` on every layer's arrivals of `iteration`."""
        s = stream if stream is not None else torch.cuda.current_stream(self.tr.device)
        _lib.call("pgx_xchg_gate_all", self.handle, iteration & 0xFFFFFFFF, s.cuda_stream)

    def join(self, layer: int, stream) -> None:
        """Make `stream` wait until this rank's part of layer's last exchange is done."""
        _lib.call("pgx_xchg_join", self.handle, layer, stream.cuda_stream)

    def check(self) -> None:
        """Raise TransportError if a bounded device wait expired (a peer died or the
        protocol wedged) — the device-side analog of finalize's watchdog (pipelined.py:60-80)."""
        status = self.tr.device_status()
        if status:
            from .errors import TransportError

            raise TransportError(f"rank {self.rank}: device wait expired (status {status}); a peer stopped "
                                 "contributing or the exchange protocol wedged")

    def launch_count(self) -> int:
        """Kernels launched by this exchange so far (exchange + gate kernels)."""
        n = C.c_uint64()
        _lib.call("pgx_xchg_launch_count", self.handle, C.byref(n))
        return n.value

    def gate(self, layer: int, iteration: int, stream=None) -> None:
        """Make `stream` (default: current) wait for layer's weights of `iteration`."""
        s = stream if stream is not None else torch.cuda.current_stream(self.tr.device)
        _lib.call("pgx_xchg_gate", self.handle, layer, iteration & 0xFFFFFFFF, s.cuda_stream)

    def close(self) -> None:
        if getattr(self, "handle", None) is not None:
            torch.cuda.synchronize(self.tr.device)
            _lib.call("pgx_xchg_destroy", self.handle)
            self.handle = None
            self._capture_keep.clear()


class ModuleBinding:
    """Drive a DeviceExchange from an nn.Module's autograd.

    `layers` is a list of (module, [params...]) in model order; layer l's flat
    vector is the concatenation of its params (W then b, like net.py:57-63).
    Parameters become views of the exchange's flat model; each layer's exchange
    launches from the post-accumulate-grad hook of its last-arriving param, on the
    exchange stream after an event on the compute stream; the module's
    forward-pre-hook gates on the previous iteration's exchange of that layer.
    """

    def __init__(self, xchg: DeviceExchange, layers, gate: str = "layer"):
        """gate="layer": each module's forward waits for its own layer (finest overlap);
        gate="model": the first forward hook of a step waits for all layers in ONE launch
        (fewer launches for many-small-layer nets; in CNNs the first layer is also the
        last one exchanged, so little overlap is lost)."""
        if gate not in ("layer", "model"):
            raise ConfigError(f"gate must be 'layer' or 'model', got {gate!r}")
        self.gate_mode = gate
        self._gated_step = None
        self.x = xchg
        self.layers = layers
        self.k = 0
        self._pending = [0] * len(layers)
        self._handles = []
        for l, (mod, params) in enumerate(layers):
            n = sum(p.numel() for p in params)
            if n != xchg.layer_elems[l]:
                raise ShapeError(f"layer {l} params hold {n} elements, exchange expects {xchg.layer_elems[l]}")
            view = xchg.layer_views[l]
            off = 0
            with torch.no_grad():
                for p in params:
                    v = view[off:off + p.numel()].view_as(p)
                    v.copy_(p.data)
                    p.data = v
                    off += p.numel()
            for p in params:
                self._handles.append(p.register_post_accumulate_grad_hook(self._make_hook(l)))
            self._handles.append(mod.register_forward_pre_hook(self._make_gate(l)))
        self.gpu_launches = 0
        self.timed_layers: set = set()   # layers whose launches are bracketed by CUDA events
        self._tstream = None
        self.trace = None                # list -> record (iteration, layer, ready_event, done_event)
        self.events: dict = {}
        self.deferred = None             # list -> phase-separated schedule: hooks queue, flush() launches
        self.disabled = False            # measurement only: hooks drop the gradients, gates pass (no exchange)

    def _make_hook(self, l):
        def hook(_p):
            if self.disabled:
                _p.grad = None
                return
            self._pending[l] += 1
            params = self.layers[l][1]
            if self._pending[l] < len(params):
                return
            self._pending[l] = 0
            if self.deferred is not None:  # barrier schedule (barrier.py:24-141): exchange after backward
                self.deferred.append((l, [p.grad if p.grad.is_contiguous() else p.grad.contiguous()
                                          for p in params]))
                for p in params:
                    p.grad = None
                return
            compute = torch.cuda.current_stream(self.x.tr.device)
            xs = self.x.stream_for(l)
            xs.wait_stream(compute)
            pieces = []
            for p in params:
                g = p.grad
                if not g.is_contiguous():
                    g = g.contiguous()
                pieces.append(g)  # DeviceExchange.launch ties their lifetime to its streams
            if self.trace is not None:  # timeline: gradient ready (compute stream) .. layer exchanged
                r0 = torch.cuda.Event(enable_timing=True)
                r0.record(compute)
            timed = l in self.timed_layers or self.trace is not None
            if timed:  # external events become event-record nodes when captured in a graph
                ext = torch.cuda.is_current_stream_capturing()
                e0 = torch.cuda.Event(enable_timing=True, external=ext)
                e1 = torch.cuda.Event(enable_timing=True, external=ext)
                e0.record(xs)
            self.x.launch(l, self.k, pieces, stream=xs)  # keeps captured pieces alive (graph lifetime)
            if timed:  # end = this rank's part done on every internal stream (copy-engine variants too)
                if self._tstream is None:
                    self._tstream = torch.cuda.Stream(device=self.x.tr.device)
                self.x.join(l, self._tstream)
                e1.record(self._tstream)
                if l in self.timed_layers:
                    self.events.setdefault(l, []).append((e0, e1))
                if self.trace is not None:
                    self.trace.append((self.k, l, r0, e1))
            for p in params:
                p.grad = None  # next backward allocates fresh gradients; the allocator
                # keeps these alive until the exchange stream is past them
            self.gpu_launches += 1
        return hook

    def _make_gate(self, l):
        def pre_hook(_mod, _inp):
            if self.disabled:
                return
            if self.gate_mode == "model":
                if self._gated_step == self.k:
                    return
                self._gated_step = self.k
                if self.x.device_iteration:
                    self.x.gate_all(-1)
                    self.gpu_launches += 1
                elif self.k > 0:
                    self.x.gate_all(self.k - 1)
                    self.gpu_launches += 1
                return
            if self.x.device_iteration:
                self.x.gate(l, -1)  # relative: the previous iteration
                self.gpu_launches += 1
            elif self.k > 0:
                self.x.gate(l, self.k - 1)
                self.gpu_launches += 1
        return pre_hook

    def flush(self) -> None:
        """Phase-separated schedule (the reference's BarrierRank, barrier.py:24-141, as the
        comparison row): launch every queued layer exchange now that backward has finished,
        in emission order, each behind the whole backward."""
        if not self.deferred:
            return
        compute = torch.cuda.current_stream(self.x.tr.device)
        for l, pieces in self.deferred:
            xs = self.x.stream_for(l)
            xs.wait_stream(compute)
            self.x.launch(l, self.k, pieces, stream=xs)
            self.gpu_launches += 1
        self.deferred.clear()

    def step_done(self) -> None:
        """Call once per iteration after backward(); raises if a device wait expired."""
        self.k += 1
        self.x.check()

    def begin_step(self) -> None:
        """Graph mode: advance the device iteration counter (capture this first)."""
        if self.x.device_iteration:
            self.x.tick()

    def drain(self) -> None:
        """Gate every layer on the last finished iteration (end of a timed region);
        in graph mode this also joins the exchange streams back for capture."""
        if self.x.device_iteration:
            cur = torch.cuda.current_stream(self.x.tr.device)
            for l in range(len(self.layers)):
                self.x.join(l, cur)
            if self._tstream is not None and torch.cuda.is_current_stream_capturing():
                cur.wait_stream(self._tstream)  # the timing stream joined the capture too
        elif self.k > 0:
            for l in range(len(self.layers)):
                self.x.gate(l, self.k - 1)

    def wait_current(self) -> None:
        """Graph mode, outside capture: wait for the latest iteration's weights everywhere."""
        for l in range(len(self.layers)):
            self.x.gate(l, 0)

    def remove(self) -> None:
        for h in self._handles:
            h.remove()
