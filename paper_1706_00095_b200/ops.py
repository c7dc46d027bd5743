"""Device versions of the path's arithmetic, same per-element expressions as the reference.

    buffer_axpy    buffers.py:69-74      y := y + alpha*x (in place, returns y)
    master_update  engine/sgd.py:27-33   w - eps*g (new tensor, inputs untouched)
    tree_reduce    engine/sgd.py:53-69   root totals of a binomial-tree fold
    fold_update    fused fold + update   (pipelined.py:158-188 + :103-108)
    seeded_fill    buffers.py:54-66      bit-identical to numpy

All take CUDA tensors and run on the current torch stream through libpgx.so.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import ShapeError
from .topology import Tree

MODES = {"ref64": _lib.MODE_REF64, "ref32": _lib.MODE_REF32, "fast32": _lib.MODE_FAST32}


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _check_cuda(*ts):
    for t in ts:
        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            raise ShapeError("device ops take CUDA tensors")
        if not t.is_contiguous():
            raise ShapeError("device ops take contiguous tensors")


def seeded_fill(seed: int, length: int, scale: float, dtype=torch.float64, device=None) -> torch.Tensor:
    if length <= 0:
        raise ShapeError(f"buffer length must be positive, got {length}")
    out = torch.empty(length, dtype=dtype, device=device or "cuda")
    fn = "pgx_seeded_fill_f64" if dtype == torch.float64 else "pgx_seeded_fill_f32"
    with torch.cuda.device(out.device):
        _lib.call(fn, seed & ((1 << 64) - 1), float(scale), out.data_ptr(), length, _stream())
    return out


def buffer_axpy(alpha: float, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    if x.shape != y.shape:
        raise ShapeError(f"axpy length mismatch: {tuple(x.shape)} vs {tuple(y.shape)}")
    if x.dtype != y.dtype:
        raise ShapeError(f"axpy dtype mismatch: {x.dtype} vs {y.dtype}")
    _check_cuda(x, y)
    fn = "pgx_axpy_f64" if y.dtype == torch.float64 else "pgx_axpy_f32"
    with torch.cuda.device(y.device):
        _lib.call(fn, float(alpha), x.data_ptr(), y.data_ptr(), y.numel(), _stream())
    return y


def master_update(weights: torch.Tensor, gradient: torch.Tensor, epsilon: float) -> torch.Tensor:
    """New tensor w - eps*g.  float64 in -> float64 out (reference-exact); float32 in ->
    the float64 result rounded to float32 (the ref32 storage rule)."""
    if weights.shape != gradient.shape:
        raise ShapeError(f"weights shape {tuple(weights.shape)} does not match gradient shape {tuple(gradient.shape)}")
    if weights.dtype != gradient.dtype:
        raise ShapeError("weights and gradient must share a dtype")
    _check_cuda(weights, gradient)
    out = torch.empty_like(weights)
    fn = "pgx_master_update_f64" if weights.dtype == torch.float64 else "pgx_master_update_f32"
    with torch.cuda.device(out.device):
        _lib.call(fn, weights.data_ptr(), gradient.data_ptr(), float(epsilon), out.data_ptr(), out.numel(), _stream())
    return out


def _ptr_array(ts):
    arr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    return arr


def tree_reduce(partials, tree, dtype=torch.float64) -> list:
    """partials[r][l] -> root totals per layer; inputs untouched.

    dtype=float64 reproduces the reference (it promotes every partial to float64,
    sgd.py:64); dtype=float32 is the ref32 fold (fp32 adds, same order)."""
    world = tree.world_size if isinstance(tree, Tree) else int(tree)
    if len(partials) != world:
        raise ShapeError(f"{len(partials)} partials for a {world}-rank tree")
    nl = len(partials[0])
    out = []
    fn = "pgx_tree_reduce_f64" if dtype == torch.float64 else "pgx_tree_reduce_f32"
    for l in range(nl):
        ts = [p[l].to(dtype).contiguous() for p in partials]
        for t in ts[1:]:
            if t.shape != ts[0].shape:
                raise ShapeError("layer partials differ in shape")
        _check_cuda(*ts)
        o = torch.empty_like(ts[0])
        with torch.cuda.device(o.device):
            _lib.call(fn, _ptr_array(ts), world, o.data_ptr(), o.numel(), _stream())
        out.append(o)
    return out


def fold_update(mode: str, partials, weights: torch.Tensor, momentum_buf: torch.Tensor | None = None, *,
                epsilon: float, scale: float = 1.0, momentum: float = 0.0, weight_decay: float = 0.0) -> torch.Tensor:
    """Fused tree-order fold of `partials` + update applied in place to `weights`."""
    m = MODES[mode]
    want = torch.float64 if m == _lib.MODE_REF64 else torch.float32
    ts = list(partials)
    for t in ts:
        if t.dtype != want or t.shape != weights.shape:
            raise ShapeError("partials must match the weights' shape and the mode's dtype")
    if weights.dtype != want:
        raise ShapeError(f"mode {mode} needs {want} weights")
    _check_cuda(weights, *ts)
    vptr = None
    if m == _lib.MODE_FAST32:
        if momentum_buf is None or momentum_buf.shape != weights.shape or momentum_buf.dtype != torch.float32:
            raise ShapeError("fast32 needs a float32 momentum buffer shaped like the weights")
        _check_cuda(momentum_buf)
        vptr = momentum_buf.data_ptr()
    with torch.cuda.device(weights.device):
        _lib.call("pgx_fold_update", m, _ptr_array(ts), len(ts), weights.data_ptr(), vptr, weights.numel(),
                  float(epsilon), float(scale), float(momentum), float(weight_decay), _stream())
    return weights
