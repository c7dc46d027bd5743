"""PSGD1 model checkpoints (reference engine/checkpoint.py:1-71) built on the device.

Same format, function names and FormatError messages as the reference:

    magic b"PSGD1"; per layer, in order: u32 index, u64 count, count x f64  (little-endian)

The image is assembled in HBM by one kernel (`pgx_ckpt_pack`: every aligned output
word from the two values it straddles — values sit at odd byte offsets), then moved
with ONE device->host copy; loading is one host->device copy plus one kernel
(`pgx_ckpt_unpack`).  Header validation (`pgx_ckpt_parse`) is host code in libpgx.
fp32 layers (the exchange's flat model) are promoted exactly to f64 on the way out,
as the reference's np.asarray(values, "<f8") does, and rounded to nearest on the way
in when the destination is fp32.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ConfigError, FormatError

MAGIC = b"PSGD1"


@dataclass
class Model:
    """A loaded checkpoint: per-layer flat device tensors (reference buffers.Model)."""

    layers: list
    iteration: int = 0


def _device(device=None) -> torch.device:
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise ConfigError("checkpoints are packed on the GPU; no CUDA device is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _flat_layers(layers, device=None) -> list:
    out = []
    dev = None
    for l, v in enumerate(layers):
        t = v if isinstance(v, torch.Tensor) else torch.as_tensor(v, dtype=torch.float64)
        if t.dim() != 1:
            raise FormatError(f"layer {l} is not a flat vector")
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if not t.is_cuda:
            dev = dev or _device(device)
            t = t.to(dev)
        out.append(t.contiguous())
    if len({t.dtype for t in out}) > 1:  # one element size per launch: promote (exact)
        out = [t.to(torch.float64) for t in out]
    return out


def image_bytes(counts) -> int:
    arr = (C.c_uint64 * max(1, len(counts)))(*counts)
    n = C.c_uint64()
    _lib.call("pgx_ckpt_image_bytes", arr, len(counts), C.byref(n))
    return n.value


def pack(layers, stream=None, out: torch.Tensor | None = None) -> tuple[torch.Tensor, int]:
    """Device image of `layers` (a uint8 CUDA tensor, padded to 16 bytes) and its length;
    `out` reuses a buffer from a previous call."""
    ts = _flat_layers(layers)
    if not ts:
        raise FormatError("checkpoint holds no layers")
    dev = ts[0].device
    counts = [t.numel() for t in ts]
    nbytes = image_bytes(counts)
    words = (nbytes + 15) // 16 * 2
    img = out.view(torch.int64) if out is not None and out.numel() >= words * 8 else \
        torch.empty(words, dtype=torch.int64, device=dev)
    ptrs = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    cnt = (C.c_uint64 * len(ts))(*counts)
    st = stream or torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):  # the launch goes to the layers' device, whatever is current
        _lib.call("pgx_ckpt_pack", ptrs, cnt, len(ts), ts[0].element_size(), C.c_void_p(img.data_ptr()),
                  words * 8, C.c_void_p(st.cuda_stream))
    return img.view(torch.uint8), nbytes


def serialize_model(layers) -> bytes:
    """PSGD1 bytes of `layers` (checkpoint.py:29-39); device tensors are packed in place."""
    layers = list(layers)
    if not layers:  # the reference writes the bare magic (and refuses to load it)
        return MAGIC
    img, nbytes = pack(layers)
    host = torch.empty(img.numel(), dtype=torch.uint8, pin_memory=True)
    host.copy_(img, non_blocking=True)
    torch.cuda.current_stream(img.device).synchronize()
    return host[:nbytes].numpy().tobytes()


def save_model(layers, path: str) -> None:
    """checkpoint.py:66-68."""
    layers = list(layers)
    if not layers:
        with open(path, "wb") as fh:
            fh.write(MAGIC)
        return
    img, nbytes = pack(layers)
    host = torch.empty(img.numel(), dtype=torch.uint8, pin_memory=True)
    host.copy_(img, non_blocking=True)
    torch.cuda.current_stream(img.device).synchronize()
    with open(path, "wb") as fh:
        fh.write(memoryview(host[:nbytes].numpy()))


def _host_view(blob):
    """(pointer, length, keep-alive) of a host byte buffer without copying it."""
    if isinstance(blob, torch.Tensor):
        return C.c_void_p(blob.data_ptr()), blob.numel() * blob.element_size(), blob
    if isinstance(blob, bytes):
        return C.cast(C.c_char_p(blob), C.c_void_p), len(blob), blob
    mv = memoryview(blob).cast("B")
    if mv.readonly:
        buf = (C.c_uint8 * max(1, len(mv))).from_buffer_copy(mv) if len(mv) else (C.c_uint8 * 1)()
    else:
        buf = (C.c_uint8 * len(mv)).from_buffer(mv) if len(mv) else (C.c_uint8 * 1)()
    return C.cast(buf, C.c_void_p), len(mv), buf


def parse(blob) -> list[int]:
    """Validate a PSGD1 blob's framing on the host; per-layer element counts."""
    ptr, nbytes, _keep = _host_view(blob)
    n = C.c_int(0)
    try:
        _lib.call("pgx_ckpt_parse", ptr, nbytes, None, 0, C.byref(n))
    except FormatError as exc:  # the reference's message, without the C-ABI function prefix
        raise FormatError(str(exc).split(": ", 1)[-1]) from None
    counts = (C.c_uint64 * n.value)()
    _lib.call("pgx_ckpt_parse", ptr, nbytes, counts, n.value, C.byref(n))
    return [int(c) for c in counts]


def _read_pinned(path: str) -> tuple[torch.Tensor, int]:
    """The file in page-locked memory (padded by a word for the unpack kernel)."""
    nbytes = os.path.getsize(path)
    host = torch.zeros(((nbytes + 7) // 8 + 1) * 8, dtype=torch.uint8, pin_memory=True)
    with open(path, "rb") as fh:
        got = fh.readinto(memoryview(host.numpy())[:nbytes])
    if got != nbytes:
        raise FormatError(f"{path}: short read ({got} of {nbytes} bytes)")
    return host, nbytes


def unpack_into(blob, layers, stream=None) -> None:
    """Decode a PSGD1 blob into existing flat device tensors (all fp32 or all fp64,
    one per layer, sizes as recorded).  `blob`: bytes-like, or a pinned uint8 tensor
    from `_read_pinned` (then `blob` is (tensor, nbytes))."""
    pinned = None
    if isinstance(blob, tuple):
        pinned, nbytes = blob
        blob = pinned[:nbytes]
    counts = parse(blob)
    if len(counts) != len(layers):
        raise FormatError(f"checkpoint holds {len(counts)} layers, model has {len(layers)}")
    for l, (n, t) in enumerate(zip(counts, layers)):
        if t.numel() != n:
            raise FormatError(f"layer {l}: checkpoint holds {n} values, model layer has {t.numel()}")
        if not (t.is_cuda and t.is_contiguous() and t.dtype in (torch.float32, torch.float64)):
            raise ConfigError(f"layer {l}: need a contiguous fp32/fp64 CUDA tensor")
    if len({t.dtype for t in layers}) > 1:
        raise ConfigError("all layers must share one dtype")
    dev = layers[0].device
    if pinned is None:
        nbytes = len(memoryview(blob).cast("B"))
        host = torch.zeros(((nbytes + 7) // 8 + 1) * 8, dtype=torch.uint8, pin_memory=True)
        host[:nbytes].copy_(torch.frombuffer(memoryview(blob).cast("B"), dtype=torch.uint8))
    else:
        host = pinned
    words = host.numel() // 8  # >= image words + 1: the last value reads one word past its own
    img = torch.empty(words * 8, dtype=torch.uint8, device=dev)
    st = stream or torch.cuda.current_stream(dev)
    with torch.cuda.stream(st):
        img.copy_(host, non_blocking=True)
    ptrs = (C.c_void_p * len(layers))(*[t.data_ptr() for t in layers])
    cnt = (C.c_uint64 * len(layers))(*counts)
    with torch.cuda.device(dev):
        _lib.call("pgx_ckpt_unpack", C.c_void_p(img.data_ptr()), words * 8, cnt, len(layers),
                  layers[0].element_size(), ptrs, C.c_void_p(st.cuda_stream))
    st.synchronize()  # the pinned staging buffer is released on return


def load_model_bytes(blob, device=None, dtype=torch.float64) -> Model:
    """checkpoint.py:42-63: validated layers as new device tensors (f64 by default, the
    reference's dtype; fp32 rounds to nearest)."""
    counts = parse(blob)
    dev = _device(device)
    layers = [torch.empty(n, dtype=dtype, device=dev) for n in counts]
    unpack_into(blob, layers)
    return Model(layers=layers, iteration=0)


def load_model(path: str, device=None, dtype=torch.float64) -> Model:
    """checkpoint.py:70-71 (the file is read straight into page-locked memory)."""
    host, nbytes = _read_pinned(path)
    counts = parse(host[:nbytes])
    dev = _device(device)
    layers = [torch.empty(n, dtype=dtype, device=dev) for n in counts]
    unpack_into((host, nbytes), layers)
    return Model(layers=layers, iteration=0)


def save_exchange(xchg, path: str) -> None:
    """Checkpoint a DeviceExchange's flat model (every layer view, in order)."""
    save_model(xchg.layer_views, path)


def load_exchange(xchg, path: str) -> None:
    """Restore a DeviceExchange's flat model from a PSGD1 file (momentum is not part of
    the format and is left as is)."""
    unpack_into(_read_pinned(path), xchg.layer_views)
