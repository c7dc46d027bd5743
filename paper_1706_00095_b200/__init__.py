"""pgx — B200-native per-layer gradient exchange (hot path of arXiv 1706.00095).

Drop-in for the reference package `pipesgd`'s exchange path: same engine surface
(PipelinedRank / BarrierRank / TrainConfig / RankResult), same transport ABI
(segment_create, write_notify, notify_poll, notify_reset, ticket_wait_all,
barrier), same arithmetic ops (buffer_axpy, master_update, tree_reduce), with the
data plane in hand-written sm_100a kernels behind the C ABI in include/pgx.h.
Importing the package does not need a GPU; calling into it does (no CPU fallback).
"""

from .config import DenseLayerSpec, TrainConfig, specs_from_dims
from .errors import (ConfigError, InputError, PipesgdError, ProtocolError, RangeError, RoutingError, ShapeError,
                     TransportError, TreeError, VerificationError)
from .layout import SEG_GRAD, SEG_MODEL, SEG_WORK, SegmentLayout
from .topology import Tree, build_broadcast_tree, build_reduction_tree, depth, fold_order, tree_check

__version__ = "0.1.0"

_LAZY = {
    "PipelinedRank": "engine", "BarrierRank": "engine", "RankResult": "engine", "TurnState": "engine",
    "batch_indices": "engine", "shard_bounds": "engine",
    "CudaTransport": "transport", "LocalWorld": "transport", "DistTransport": "transport",
    "WriteRequest": "transport", "Ticket": "transport", "LatencyModel": "transport", "CONTROL_SEGMENT": "transport",
    "buffer_axpy": "ops", "master_update": "ops", "tree_reduce": "ops", "fold_update": "ops", "seeded_fill": "ops",
    "DeviceExchange": "exchange", "ModuleBinding": "exchange",
    "run_local": "harness", "run_dist": "harness", "sequential_sgd": "harness",
    "verify_against_reference": "harness", "build_dataset": "harness",
    "Recorder": "timeline", "compute_overlap": "timeline", "TimelineEvent": "timeline", "RunMetrics": "timeline",
    "read_timeline_csv": "timeline", "write_timeline_csv": "timeline",
    "serialize_model": "checkpoint", "load_model_bytes": "checkpoint", "save_model": "checkpoint",
    "load_model": "checkpoint", "Model": "checkpoint", "save_exchange": "checkpoint", "load_exchange": "checkpoint",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted(list(_LAZY) + [
    "DenseLayerSpec", "TrainConfig", "specs_from_dims", "ConfigError", "InputError", "PipesgdError",
    "ProtocolError", "RangeError", "RoutingError", "ShapeError", "TransportError", "TreeError",
    "VerificationError", "SEG_GRAD", "SEG_MODEL", "SEG_WORK", "SegmentLayout", "Tree", "build_broadcast_tree",
    "build_reduction_tree", "depth", "fold_order", "tree_check"])
