"""ctypes binding of libpgx.so (include/pgx.h).

The product path has no fallback: if the shared library is missing or fails to
load, every entry point raises immediately.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_1706_00095_b200/csrc``).
"""

from __future__ import annotations

import ctypes as C
import os
import re

from .errors import TransportError, raise_for

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpgx.so")
HEADER_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "pgx.h")

IPC_HANDLE_BYTES = 64
CONTROL_SEGMENT = 15
MAX_RANKS = 8
MAX_PIECES = 4
XCHG_STREAMS = 5
CKPT_MAX_LAYERS = 512

MODE_REF64, MODE_REF32, MODE_FAST32, MODE_SUM32 = 0, 1, 2, 3
VARIANT_TREE, VARIANT_TWOSHOT, VARIANT_TWOSHOT_CE, VARIANT_NVLS, VARIANT_ONESHOT = 0, 1, 2, 3, 4
VARIANT_TWOSHOT_CEP = 5
VARIANT_ONESHOT_LL = 6
VARIANT_ONESHOT_L128 = 7
VARIANT_TWOSHOT_BULK = 8
VARIANT_TWOSHOT_L128 = 9
XF_CE_RS_PARTS, XF_TMA, XF_ONESHOT_SMALL_CHUNKS, XF_AUTO_CHUNK_TREE, XF_NO_AUTO_CHUNK_NVLS, XF_ALLOW_L128 = 1, 2, 4, 8, 16, 32
XF_BULK_LEAN = 64
XF_BULK_CE_RS = 128
XF_CE_TMA_OWNER = 256
XF_LEAN_CAPPED = 512
PHASE_PUSH, PHASE_OWNER, PHASE_DOWN, PHASE_ALL = 1, 2, 4, 7

vp = C.c_void_p
u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int
P = C.POINTER


class XchgConfig(C.Structure):
    _fields_ = [
        ("num_layers", i32),
        ("layer_elems", P(u64)),
        ("variant", P(i32)),
        ("mode", i32),
        ("chunk_elems", u64),
        ("lr", C.c_double),
        ("scale", C.c_float),
        ("momentum", C.c_float),
        ("weight_decay", C.c_float),
        ("seg_base", u32),
        ("max_ctas", i32),
        ("layer_chunk_elems", P(u64)),
        ("layer_max_ctas", P(i32)),
        ("ce_parts", i32),
        ("ce_rs_streams", i32),
        ("flags", u32),
    ]


# name -> argtypes (restype is always int unless listed in _RESTYPE)
SIGNATURES = {
    "pgx_abi_version": [],
    "pgx_last_error": [],
    "pgx_world_create": [i32, i32, i32, P(vp)],
    "pgx_world_destroy": [vp],
    "pgx_world_status": [vp, P(u32)],
    "pgx_world_clear_status": [vp],
    "pgx_world_set_timeout": [vp, C.c_double],
    "pgx_segment_create": [vp, u32, u64, u32, P(vp), P(vp)],
    "pgx_segment_info": [vp, i32, u32, P(vp), P(vp), P(u64), P(u32)],
    "pgx_segment_export": [vp, u32, vp],
    "pgx_segment_attach_ipc": [vp, i32, u32, vp, u64, u32],
    "pgx_segment_attach_local": [vp, i32, u32, vp, vp, u64, u32],
    "pgx_enable_peer_access": [i32, i32],
    "pgx_write_notify": [vp, u32, u64, i32, u32, u64, u64, u32, u32, vp],
    "pgx_write_notify_chunked": [vp, u32, u64, i32, u32, u64, u64, u64, u32, u32, vp],
    "pgx_notify_poll": [vp, u32, u32, u32, P(u32), P(u32), u32, P(u32)],
    "pgx_notify_reset": [vp, u32, u32, P(u32)],
    "pgx_ticket_record": [vp, P(vp)],
    "pgx_ticket_query": [vp],
    "pgx_ticket_wait": [vp, C.c_double],
    "pgx_ticket_release": [vp],
    "pgx_barrier": [vp, vp, C.c_double],
    "pgx_barrier_async": [vp, vp, C.c_double],
    "pgx_axpy_f64": [C.c_double, vp, vp, u64, vp],
    "pgx_axpy_f32": [C.c_float, vp, vp, u64, vp],
    "pgx_master_update_f64": [vp, vp, C.c_double, vp, u64, vp],
    "pgx_master_update_f32": [vp, vp, C.c_double, vp, u64, vp],
    "pgx_tree_reduce_f64": [P(vp), i32, vp, u64, vp],
    "pgx_tree_reduce_f32": [P(vp), i32, vp, u64, vp],
    "pgx_fold_update": [i32, P(vp), i32, vp, vp, u64, C.c_double, C.c_float, C.c_float, C.c_float, vp],
    "pgx_ckpt_image_bytes": [P(u64), i32, P(u64)],
    "pgx_ckpt_parse": [vp, u64, P(u64), i32, P(i32)],
    "pgx_ckpt_pack": [P(vp), P(u64), i32, i32, vp, u64, vp],
    "pgx_ckpt_unpack": [vp, u64, P(u64), i32, i32, P(vp), vp],
    "pgx_seeded_fill_f64": [u64, C.c_double, vp, u64, vp],
    "pgx_seeded_fill_f32": [u64, C.c_double, vp, u64, vp],
    "pgx_xchg_create": [vp, P(XchgConfig), P(vp)],
    "pgx_xchg_destroy": [vp],
    "pgx_xchg_model": [vp, P(vp), P(u64)],
    "pgx_xchg_connect": [vp],
    "pgx_xchg_layer": [vp, i32, u32, P(vp), P(u64), i32, i32, vp],
    "pgx_xchg_gate": [vp, i32, u32, vp],
    "pgx_xchg_gate_all": [vp, u32, vp],
    "pgx_xchg_nvls_export": [vp, P(i32)],
    "pgx_xchg_nvls_import": [vp, i32],
    "pgx_xchg_nvls_bind": [vp],
    "pgx_xchg_layer_bytes": [vp, i32, P(u64), P(u64)],
    "pgx_xchg_layer_plan": [vp, i32, P(u64), P(i32)],
    "pgx_xchg_layer_parts": [vp, i32, P(i32)],
    "pgx_xchg_set_trace": [vp, vp],
    "pgx_graph_instantiate_prio": [vp, P(vp)],
    "pgx_graph_launch": [vp, vp],
    "pgx_graph_exec_destroy": [vp],
    "pgx_xchg_launch_count": [vp, P(u64)],
    "pgx_xchg_stream": [vp, i32, P(vp)],
    "pgx_xchg_set_streams": [vp, P(vp), i32],
    "pgx_xchg_join": [vp, i32, vp],
    "pgx_xchg_device_iteration": [vp, i32, u32],
    "pgx_xchg_tick": [vp, vp],
}
_RESTYPE = {"pgx_last_error": C.c_char_p}

_lib = None


def header_symbols() -> list[str]:
    """Every function the C header declares (the ABI contract)."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(pgx_\w+)\s*\(", text, re.M)))


def lib():
    """The loaded library; raises TransportError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise TransportError(f"libpgx.so is not built ({LIB_PATH}); run __graft_entry__.build()")
    try:
        handle = C.CDLL(LIB_PATH)
    except OSError as exc:
        raise TransportError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, argtypes in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPE.get(name, C.c_int)
    _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().pgx_last_error()
    return msg.decode() if msg else ""


def call(name: str, *args) -> int:
    """Invoke one C-ABI function; nonzero status raises the mapped exception."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise_for(rc, f"{name}: {last_error()}")
    return rc


def stream_ptr(stream) -> int | None:
    """cudaStream_t of a torch.cuda.Stream (None -> legacy default stream)."""
    if stream is None:
        return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
