"""CPU oracle for the per-layer gradient-exchange path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the arithmetic and bookkeeping of the
reference's hot path (`pipesgd`, /root/reference/pkg/src/pipesgd).  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it, and only as the checker; the product
path (`paper_1706_00095_b200`) never imports anything under `oracle/`.

Pinning: every function here is checked against golden vectors produced by
running the reference package itself (`tests/golden/make_golden.py`, committed
fixtures `tests/golden/golden.{npz,json}`), see `tests/test_oracle_golden.py`.
The fast32 (momentum / weight decay / 1/N) rule has no counterpart in the
reference — it restates Caffe's SGDSolver and is marked
"parity unpinned" below.

Citations are `file:line` relative to /root/reference/pkg/src/pipesgd/.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
MIX_A = 0xBF58476D1CE4E5B9
MIX_B = 0x94D049BB133111EB
F64_BYTES = 8  # engine/layout.py:35


# ----------------------------------------------------------------------------- PRNG
def mix64(z: int) -> int:
    """splitmix64 finalizer (buffers.py:23-28)."""
    z &= M64
    z = ((z ^ (z >> 30)) * MIX_A) & M64
    z = ((z ^ (z >> 27)) * MIX_B) & M64
    return z ^ (z >> 31)


def derived_seed(seed: int, *tags: int) -> int:
    """Tag folding: state = mix64(state ^ mix64(tag)) per tag (buffers.py:31-36)."""
    s = seed & M64
    for t in tags:
        s = mix64(s ^ mix64(t & M64))
    return s


def splitmix64_stream(seed: int, count: int) -> np.ndarray:
    """n-th output = mix64(seed + (n+1)*GAMMA), wrapping uint64 (buffers.py:39-51)."""
    n = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & M64) + n * np.uint64(GOLDEN_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX_A)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX_B)
    return z ^ (z >> np.uint64(31))


def seeded_fill(seed: int, length: int, scale: float) -> np.ndarray:
    """scale * (2u - 1), u = top 53 bits / 2^53 (buffers.py:54-66)."""
    z = splitmix64_stream(seed, length)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return scale * (2.0 * u - 1.0)


# ----------------------------------------------------------------------------- trees
def tree_parent(r: int) -> int:
    """parent(r) = r with its lowest set bit cleared (topology.py:40-41)."""
    return r & (r - 1)


def tree_children(r: int, world: int) -> list[int]:
    """Children of r, ascending (topology.py:42-44): c = r + j for j = 1,2,4,.. below lowbit(r)."""
    out = []
    low = (r & -r) if r else 1 << 62
    j = 1
    while j < low and r + j < world:
        out.append(r + j)
        j <<= 1
    return out


def tree_depth(world: int) -> int:
    """Longest root-to-leaf path (topology.py:58-68)."""
    return max((bin(r).count("1") for r in range(world)), default=0)


# ----------------------------------------------------------------------------- arithmetic
def buffer_axpy(alpha: float, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """y := y + (alpha * x), two roundings, dtype of y kept (buffers.py:69-74)."""
    if x.shape != y.shape:
        raise ValueError("shape mismatch")
    y += alpha * x
    return y


def master_update(w: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """w - eps*g computed in float64, inputs promoted, new array (sgd.py:27-33)."""
    w64 = np.asarray(w, dtype=np.float64)
    g64 = np.asarray(g, dtype=np.float64)
    return w64 - eps * g64


def master_update_ref32(w32: np.ndarray, g32: np.ndarray, eps: float) -> np.ndarray:
    """ref32 storage rule: the reference update on fp32 arrays, result stored as fp32."""
    return master_update(w32, g32, eps).astype(np.float32)


def tree_reduce(partials, world: int, dtype=np.float64) -> list[np.ndarray]:
    """Fold per-rank partials up the binomial tree (sgd.py:53-69).

    dtype=float64 is the reference's tree_reduce (it copies inputs as float64,
    sgd.py:64).  dtype=float32 is the `ref32` convention: the reference's
    buffer_axpy applied to fp32 arrays in the same order.
    """
    acc = [[np.array(v, dtype=dtype, copy=True) for v in pr] for pr in partials]
    for r in range(world - 1, -1, -1):
        for c in tree_children(r, world):
            for l in range(len(acc[r])):
                buffer_axpy(1.0, acc[c][l], acc[r][l])
    return acc[0]


def fast32_update(w: np.ndarray, v: np.ndarray, g_sum: np.ndarray, scale: float, lr: float,
                  momentum: float, weight_decay: float):
    """fast32 rule — PARITY UNPINNED (no reference counterpart).

    Restates Caffe SGDSolver (external, BVLC caffe sgd_solver.cpp Regularize +
    ComputeUpdateValue + Blob::Update), evaluated in fp32 with one rounding per
    operation and no FMA contraction, in this order:
        g = scale*g_sum ; g = g + wd*w ; v = mu*v + lr*g ; w = w - v
    Returns (w_new, v_new) as float32.
    """
    f = np.float32
    g = (f(scale) * g_sum.astype(f)).astype(f)
    g = (g + (f(weight_decay) * w.astype(f)).astype(f)).astype(f)
    v_new = ((f(momentum) * v.astype(f)).astype(f) + (f(lr) * g).astype(f)).astype(f)
    w_new = (w.astype(f) - v_new).astype(f)
    return w_new, v_new


# ----------------------------------------------------------------------------- layout
def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


class Layout:
    """Segment offsets / notification-id blocks (engine/layout.py:42-139).

    elem_bytes generalises the reference's fixed 8-byte floats (layout.py:35)
    so the same rules describe fp32 segments; with elem_bytes=8 every number
    equals the reference's.
    """

    def __init__(self, counts, chunk_bytes: int, elem_bytes: int = F64_BYTES):
        self.counts = list(counts)
        self.L = len(counts)
        self.chunk_bytes = chunk_bytes
        self.layer_bytes = [c * elem_bytes for c in counts]
        self.layer_offsets = list(np.cumsum([0] + self.layer_bytes[:-1]).astype(int))
        self.total_bytes = int(sum(self.layer_bytes))
        self.layer_chunks = [ceil_div(b, chunk_bytes) for b in self.layer_bytes]
        self.max_chunks = max(self.layer_chunks)
        self.bulk_chunks = ceil_div(self.total_bytes, chunk_bytes)
        self.blk = self.max_chunks + 1
        self.bblk = self.bulk_chunks + 1

    def model_notif_base(self, l, p):
        return 1 + (2 * l + p) * self.blk

    def grad_notif_base(self, c, l, p):
        return 1 + c * self.L * 2 * self.blk + (2 * l + p) * self.blk

    def model_bulk_base(self, p):
        return 1 + self.L * 2 * self.blk + p * self.bblk

    def grad_bulk_base(self, nc, c, p):
        return 1 + nc * self.L * 2 * self.blk + (2 * c + p) * self.bblk

    def model_notif_count(self):
        return 1 + self.L * 2 * self.blk + 2 * self.bblk

    def grad_notif_count(self, nc):
        n = max(1, nc)
        return 1 + n * self.L * 2 * self.blk + n * 2 * self.bblk

    def model_slot_offset(self, l, p):
        return p * self.total_bytes + self.layer_offsets[l]

    def grad_slot_offset(self, c, l, p):
        return (2 * c + p) * self.total_bytes + self.layer_offsets[l]

    @staticmethod
    def chunk_id(base, j, n):
        """Final chunk carries the base id, earlier ones base+1+j (layout.py:130-139)."""
        return base if j == n - 1 else base + 1 + j


# ----------------------------------------------------------------------------- batches
TAG_BATCH = 0x6261746368  # engine/sgd.py:24


def batch_indices(seed: int, k: int, batch: int, dataset: int) -> np.ndarray:
    """splitmix stream keyed on (seed, TAG_BATCH, k) mod dataset size (sgd.py:36-44)."""
    s = splitmix64_stream(derived_seed(seed, TAG_BATCH, k), batch)
    return (s % np.uint64(dataset)).astype(np.int64)


def shard_bounds(batch: int, world: int, rank: int):
    """Contiguous [lo, hi) of rank's shard (sgd.py:47-50)."""
    sh = batch // world
    return rank * sh, (rank + 1) * sh


# ----------------------------------------------------------------------------- exchange
def exchange_iteration(grads, weights, eps: float, mode: str = "ref32", state=None,
                       scale=1.0, lr=None, momentum=0.0, weight_decay=0.0):
    """One full exchange of one layer: tree reduce -> update -> broadcast.

    grads[r] is rank r's local gradient for the layer, `weights` the model before
    the update.  Returns the updated weights every rank must hold afterwards
    (pipelined.py:158-203 fold/complete/arrival; sgd.py:27-33 update).
    """
    world = len(grads)
    if mode == "ref64":
        red = tree_reduce([[g] for g in grads], world, np.float64)[0]
        return master_update(weights, red, eps)
    if mode == "ref32":
        red = tree_reduce([[g] for g in grads], world, np.float32)[0]
        return master_update_ref32(weights, red, eps)
    if mode == "fast32":
        red = tree_reduce([[g] for g in grads], world, np.float32)[0]
        v = state if state is not None else np.zeros_like(weights, dtype=np.float32)
        return fast32_update(weights, v, red, scale, eps if lr is None else lr, momentum, weight_decay)
    if mode == "sum32":  # update off: the averaged all-reduce result, fl(scale * tree_sum) (no reference counterpart)
        red = tree_reduce([[g] for g in grads], world, np.float32)[0]
        return (np.float32(scale) * red).astype(np.float32)
    raise ValueError(mode)


# ----------------------------------------------------------------------------- formats
CKPT_MAGIC = b"PSGD1"  # engine/checkpoint.py:23


class CheckpointFormatError(ValueError):
    """Oracle-side stand-in for the reference's FormatError (errors.py:49)."""


def ckpt_serialize(layers) -> bytes:
    """PSGD1 image (engine/checkpoint.py:29-39): magic, then per layer little-endian
    u32 index, u64 count and the values as '<f8' (fp32 promoted exactly)."""
    parts = [CKPT_MAGIC]
    for l, values in enumerate(layers):
        a = np.ascontiguousarray(values, dtype="<f8")
        if a.ndim != 1:
            raise CheckpointFormatError(f"layer {l} is not a flat vector")
        parts.append(np.array([l], "<u4").tobytes() + np.array([a.size], "<u8").tobytes())
        parts.append(a.tobytes())
    return b"".join(parts)


def ckpt_load(blob: bytes) -> list:
    """Walk and validate a PSGD1 image (engine/checkpoint.py:42-63), same checks and
    messages in the same order; returns the f64 layers."""
    if blob[:5] != CKPT_MAGIC:
        raise CheckpointFormatError(f"bad checkpoint magic {blob[:5]!r}")
    pos, out = 5, []
    while pos < len(blob):
        if len(blob) - pos < 12:
            raise CheckpointFormatError("truncated checkpoint: partial layer header")
        index = int(np.frombuffer(blob, "<u4", 1, pos)[0])
        count = int(np.frombuffer(blob, "<u8", 1, pos + 4)[0])
        pos += 12
        if index != len(out):
            raise CheckpointFormatError(f"layer {len(out)} recorded with index {index}")
        if pos + 8 * count > len(blob):
            raise CheckpointFormatError(f"truncated checkpoint: layer {index} shorter than declared")
        out.append(np.frombuffer(blob, "<f8", count, pos).astype(np.float64))
        pos += 8 * count
    if not out:
        raise CheckpointFormatError("checkpoint holds no layers")
    return out


def overlap_metrics(events):
    """Run metrics of a timeline (timeline.py:137-175). events: (rank, iteration, layer,
    kind, t0, t1).  Per rank: sum over COMM events of |event ∩ union(COMPUTE)| over the sum
    of COMM lengths; averaged over ranks that communicated; wall clock per rank; run
    iterations/s = (max iteration + 1) / span."""
    comm_k = {"send_trigger", "recv_notify", "model_forward"}
    comp_k = {"forward", "backward_layer", "reduce_local", "master_update"}
    ranks = sorted({e[0] for e in events})
    ratios, wall, per = [], {}, {}
    for r in ranks:
        ev = [e for e in events if e[0] == r]
        spans = sorted((e[4], e[5]) for e in ev if e[3] in comp_k)
        union = []
        for a, b in spans:
            if union and a <= union[-1][1]:
                union[-1][1] = max(union[-1][1], b)
            else:
                union.append([a, b])
        tot = hid = 0
        for e in ev:
            if e[3] in comm_k:
                tot += e[5] - e[4]
                hid += sum(max(0, min(e[5], hi) - max(e[4], lo)) for lo, hi in union)
        wall[r] = max(e[5] for e in ev) - min(e[4] for e in ev)
        if tot > 0:
            per[r] = hid / tot
            ratios.append(hid / tot)
    ips = 0.0
    if events:
        span = max(e[5] for e in events) - min(e[4] for e in events)
        if span > 0:
            ips = (max(e[1] for e in events) + 1) / (span * 1e-9)
    return {"overlap_ratio": sum(ratios) / len(ratios) if ratios else 0.0, "iterations_per_second": ips,
            "wall_clock_ns": wall, "per_rank_overlap": per}
