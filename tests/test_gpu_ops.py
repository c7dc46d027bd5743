"""Device arithmetic vs the CPU oracle / reference golden vectors (bit-exact)."""

import numpy as np
import pytest
import torch

from oracle import pipesgd_oracle as O

pytestmark = pytest.mark.gpu

LENET = [520, 25050, 400500, 5010]
CIFAR = [2432, 25632, 51264, 65600, 650]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def test_seeded_fill_is_bit_identical(cuda, golden):
    from paper_1706_00095_b200.ops import seeded_fill

    arr, meta = golden
    for i, (s, n, sc) in enumerate(meta["fills"]):
        assert host(seeded_fill(int(s), n, sc)).tobytes() == arr[f"fill_{i}"].tobytes()
    big = host(seeded_fill(12345, 1 << 20, 0.1))
    assert big.tobytes() == O.seeded_fill(12345, 1 << 20, 0.1).tobytes()
    f32 = host(seeded_fill(7, 1001, 1.0, torch.float32))
    assert f32.tobytes() == O.seeded_fill(7, 1001, 1.0).astype(np.float32).tobytes()


def test_buffer_axpy_golden_and_property(cuda, golden):
    from paper_1706_00095_b200.ops import buffer_axpy

    arr, meta = golden
    y = dev(np.array([1.0, 2.0, 3.0]))
    out = buffer_axpy(2.0, dev(np.array([10.0, 20.0, 30.0])), y)
    assert out is y and host(y).tolist() == [21.0, 42.0, 63.0]
    for i, a in enumerate(meta["axpy_alphas"]):
        y = dev(arr["axpy_y0"])
        buffer_axpy(a, dev(arr["axpy_x"]), y)
        assert host(y).tobytes() == arr[f"axpy_out_{i}"].tobytes()
    y = dev(arr["axpy_y0"].astype(np.float32))
    buffer_axpy(1.0, dev(arr["axpy_x"].astype(np.float32)), y)
    assert host(y).tobytes() == arr["axpy32_out"].tobytes()


@pytest.mark.parametrize("n", [1, 3, 4, 5, 17, 25050, 400500, (1 << 22) + 3])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("offset", [0, 1])
def test_axpy_sizes_and_misaligned_views(cuda, n, dtype, offset):
    from paper_1706_00095_b200.ops import buffer_axpy

    rng = np.random.default_rng(n)
    x = rng.normal(size=n + offset).astype(dtype) * 1e3
    y = rng.normal(size=n + offset).astype(dtype)
    dx, dy = dev(x), dev(y)
    buffer_axpy(-0.37, dx[offset:], dy[offset:])
    want = y.copy()
    O.buffer_axpy(dtype(-0.37) if dtype == np.float32 else -0.37, x[offset:], want[offset:])
    assert host(dy).tobytes() == want.tobytes()


def test_master_update_golden(cuda, golden):
    from paper_1706_00095_b200.ops import master_update

    arr, meta = golden
    out = master_update(dev(np.array([1.0, 0.0, -1.0])), dev(np.array([0.2, 0.0, -0.2])), 0.5)
    assert host(out).tolist() == [0.9, 0.0, -0.9]
    w, g = dev(arr["upd_w"]), dev(arr["upd_g"])
    for i, eps in enumerate(meta["upd_eps"]):
        assert host(master_update(w, g, eps)).tobytes() == arr[f"upd_out_{i}"].tobytes()
    assert host(w).tobytes() == arr["upd_w"].tobytes()  # inputs untouched
    o32 = master_update(dev(arr["upd_w"].astype(np.float32)), dev(arr["upd_g"].astype(np.float32)), 0.05)
    assert host(o32).tobytes() == arr["upd32_out"].astype(np.float32).tobytes()


@pytest.mark.parametrize("s", range(1, 9))
def test_tree_reduce_matches_reference_golden(cuda, golden, s):
    from paper_1706_00095_b200.ops import tree_reduce

    arr, _ = golden
    parts = [[dev(arr[f"tr{s}_in_{r}_0"]), dev(arr[f"tr{s}_in_{r}_1"])] for r in range(s)]
    out = tree_reduce(parts, s)
    assert host(out[0]).tobytes() == arr[f"tr{s}_out_0"].tobytes()
    assert host(out[1]).tobytes() == arr[f"tr{s}_out_1"].tobytes()
    p32 = [[p[0].float()] for p in parts]
    assert host(tree_reduce(p32, s)[0]).tobytes() == arr[f"tr{s}_out32_0"].tobytes()
    assert host(tree_reduce(p32, s, dtype=torch.float32)[0]).tobytes() == arr[f"tr{s}_ref32_0"].tobytes()


def test_fold_order_cancellation_on_device(cuda):
    from paper_1706_00095_b200.ops import tree_reduce

    parts = [[dev(np.full(5, v))] for v in (1e16, 1.0, -1e16, 0.0)]
    assert host(tree_reduce(parts, 4)[0]).tolist() == [0.0] * 5


@pytest.mark.parametrize("s", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("n", LENET + CIFAR[:2])
@pytest.mark.parametrize("mode", ["ref64", "ref32", "fast32"])
def test_fused_fold_update_vs_oracle(cuda, s, n, mode):
    from paper_1706_00095_b200.ops import fold_update

    dt = np.float64 if mode == "ref64" else np.float32
    grads = [O.seeded_fill(O.derived_seed(42, r, n), n, 1e-3).astype(dt) for r in range(s)]
    w = O.seeded_fill(42 ^ 5, n, 1 / np.sqrt(n)).astype(dt)
    v = O.seeded_fill(99, n, 1e-4).astype(np.float32)
    dw, dv = dev(w), dev(v)
    fold_update(mode, [dev(g) for g in grads], dw, dv if mode == "fast32" else None, epsilon=0.01, scale=1.0 / s,
                momentum=0.9, weight_decay=5e-4)
    if mode == "fast32":
        want_w, want_v = O.exchange_iteration(grads, w, 0.01, mode, state=v, scale=1.0 / s, momentum=0.9,
                                              weight_decay=5e-4)
        got_w, got_v = host(dw), host(dv)
        np.testing.assert_allclose(got_w, want_w, rtol=1e-5, atol=0)   # the north-star tolerance
        assert got_w.tobytes() == want_w.tobytes() and got_v.tobytes() == want_v.tobytes()  # and in fact exact
    else:
        want = O.exchange_iteration(grads, w, 0.01, mode)
        assert host(dw).tobytes() == want.astype(dt).tobytes()
