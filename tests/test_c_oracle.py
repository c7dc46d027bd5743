"""The C restatement (timed CPU port) agrees with the numpy oracle and the reference."""

import numpy as np
import pytest

from oracle import c_oracle as CO
from oracle import pipesgd_oracle as O


@pytest.mark.parametrize("s", range(1, 9))
def test_c_fold_matches_reference_golden(golden, s):
    arr, _ = golden
    parts = [arr[f"tr{s}_in_{r}_0"] for r in range(s)]
    assert CO.tree_fold(parts).tobytes() == arr[f"tr{s}_out_0"].tobytes()
    p32 = [p.astype(np.float32) for p in parts]
    assert CO.tree_fold(p32).tobytes() == arr[f"tr{s}_ref32_0"].tobytes()


def test_c_updates_match_numpy_oracle(golden):
    arr, _ = golden
    w, g = arr["upd_w"].astype(np.float32), arr["upd_g"].astype(np.float32)
    assert CO.update_ref32(w, g, 0.05).tobytes() == O.master_update_ref32(w, g, 0.05).tobytes()
    v = np.linspace(-1, 1, w.size).astype(np.float32)
    a = CO.update_fast32(w, v, g, 0.25, 0.01, 0.9, 5e-4)
    b = O.fast32_update(w, v, g, 0.25, 0.01, 0.9, 5e-4)
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("threads", [1, 3])
def test_c_exchange_port_matches_oracle(world, threads):
    elems = [520, 25050, 5010]
    ex = CO.ExchangeWorld(world, elems)
    grads = [[g.copy() for g in ex.grad[r]] for r in range(world)]
    w0 = [a.copy() for a in ex.w[0]]
    ex.iteration("fast32", lr=0.01, mu=0.9, wd=5e-4, threads=threads)
    for l in range(len(elems)):
        want, _ = O.exchange_iteration([grads[r][l] for r in range(world)], w0[l], 0.01, "fast32",
                                       state=np.zeros(elems[l], np.float32), scale=1.0 / world, momentum=0.9,
                                       weight_decay=5e-4)
        for r in range(world):
            assert ex.w[r][l].tobytes() == want.tobytes()


@pytest.mark.parametrize("mode", ["ref32", "sum32"])
def test_c_exchange_port_other_modes(mode):
    elems = [520, 25050, 5010]
    world = 4
    ex = CO.ExchangeWorld(world, elems)
    grads = [[g.copy() for g in ex.grad[r]] for r in range(world)]
    w0 = [a.copy() for a in ex.w[0]]
    ex.iteration(mode, lr=0.05, threads=2)
    for l in range(len(elems)):
        kw = {"scale": 1.0 / world} if mode == "sum32" else {}
        want = O.exchange_iteration([grads[r][l] for r in range(world)], w0[l], 0.05, mode, **kw)
        for r in range(world):
            assert ex.w[r][l].tobytes() == np.asarray(want, np.float32).tobytes()
