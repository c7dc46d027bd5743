"""ctypes wrapper of oracle/build/liboracle.so — TEST / BASELINE INFRASTRUCTURE ONLY.

Used by tests (checked against the numpy oracle and the reference golden vectors)
and by bench.py's cpu_baseline / --impl reference legs as the timed CPU port of
the reference's exchange data plane.  Never imported by the product package.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "build", "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} not built (make -C oracle)")
        _lib = C.CDLL(LIB)
        P = C.POINTER
        _lib.oracle_tree_fold_f32.argtypes = [P(C.c_void_p), C.c_int, C.c_void_p, C.c_size_t]
        _lib.oracle_tree_fold_f64.argtypes = [P(C.c_void_p), C.c_int, C.c_void_p, C.c_size_t]
        _lib.oracle_update_ref32.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_size_t]
        _lib.oracle_update_ref64.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_size_t]
        _lib.oracle_update_fast32.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_float, C.c_float,
                                              C.c_float, C.c_size_t]
        _lib.oracle_exchange_iteration.argtypes = [C.c_int, C.c_int, P(C.c_uint64), C.c_void_p, C.c_void_p,
                                                   C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_float,
                                                   C.c_float, C.c_float, C.c_int]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def tree_fold(parts):
    parts = [np.ascontiguousarray(p) for p in parts]
    out = np.empty_like(parts[0])
    ptrs = (C.c_void_p * len(parts))(*[p.ctypes.data for p in parts])
    fn = lib().oracle_tree_fold_f64 if out.dtype == np.float64 else lib().oracle_tree_fold_f32
    fn(ptrs, len(parts), _p(out), out.size)
    return out


def update_ref32(w, g, eps):
    w = w.astype(np.float32).copy()
    lib().oracle_update_ref32(_p(w), _p(np.ascontiguousarray(g, np.float32)), eps, w.size)
    return w


def update_fast32(w, v, g, scale, lr, mu, wd):
    w = w.astype(np.float32).copy()
    v = v.astype(np.float32).copy()
    lib().oracle_update_fast32(_p(w), _p(v), _p(np.ascontiguousarray(g, np.float32)), scale, lr, mu, wd, w.size)
    return w, v


class ExchangeWorld:
    """fp32 buffers of `world` ranks for the CPU port of one pipelined iteration."""

    def __init__(self, world: int, elems, seed: int = 42, fast_fill: bool = False):
        """fast_fill: numpy PCG64 draws instead of seeded_fill (timing runs at full model
        sizes, where the arithmetic does not depend on the values and seeded_fill's
        splitmix stream in numpy would take ~25 s for 8 AlexNet gradients)."""
        from . import pipesgd_oracle as O

        self.world, self.elems = world, [int(n) for n in elems]
        L = len(self.elems)
        if fast_fill:
            rng = np.random.default_rng(seed)

            def fill(_s, n, scale):
                return (rng.standard_normal(n, dtype=np.float32) * np.float32(scale)).astype(np.float32)
        else:
            def fill(s, n, scale):
                return O.seeded_fill(s, n, scale).astype(np.float32)
        self.grad = [[fill(O.derived_seed(seed, r, l), n, 1e-3) for l, n in enumerate(self.elems)]
                     for r in range(world)]
        w0 = [fill(seed ^ l, n, 0.01) for l, n in enumerate(self.elems)]
        self.w = [[a.copy() for a in w0] for _ in range(world)]
        self.v = [np.zeros(n, np.float32) for n in self.elems]
        self.rx = [[np.zeros(n, np.float32) for n in self.elems] for _ in range(world)]
        self._keep = []

        def table(rows):
            outer = (C.c_void_p * len(rows))()
            for i, row in enumerate(rows):
                inner = (C.c_void_p * L)(*[a.ctypes.data for a in row])
                self._keep.append(inner)
                outer[i] = C.cast(inner, C.c_void_p)
            self._keep.append(outer)
            return outer

        self._g, self._w, self._rx = table(self.grad), table(self.w), table(self.rx)
        self._v = (C.c_void_p * L)(*[a.ctypes.data for a in self.v])
        self._e = (C.c_uint64 * L)(*self.elems)

    def iteration(self, mode="fast32", lr=0.01, scale=None, mu=0.9, wd=5e-4, threads=1):
        m = {"ref32": 1, "fast32": 2, "sum32": 3}[mode]
        sc = 1.0 / self.world if scale is None else scale
        lib().oracle_exchange_iteration(self.world, len(self.elems), self._e, C.cast(self._g, C.c_void_p),
                                        C.cast(self._w, C.c_void_p), C.cast(self._v, C.c_void_p),
                                        C.cast(self._rx, C.c_void_p), m, lr, sc, mu, wd, threads)

    @property
    def bytes_per_iteration(self) -> int:
        return 4 * sum(self.elems)
