"""The CPU oracle (oracle/pipesgd_oracle.py) pinned against the reference's own outputs.

Golden vectors come from running the reference package (tests/golden/make_golden.py);
these tests check every oracle function the parity tests rely on.
"""

import numpy as np
import pytest

from oracle import pipesgd_oracle as O


def test_splitmix_streams(golden):
    arr, meta = golden
    for i, s in enumerate(meta["splitmix_seeds"]):
        assert np.array_equal(O.splitmix64_stream(int(s), 17), arr[f"splitmix_{i}"])


def test_mix64_and_derived_seed(golden):
    _, meta = golden
    for z, want in meta["mix64"].items():
        assert O.mix64(int(z)) == int(want)
    for seed, tags, want in meta["derived_seed"]:
        assert O.derived_seed(int(seed), *tags) == int(want)


def test_seeded_fill_bits(golden):
    arr, meta = golden
    for i, (s, n, sc) in enumerate(meta["fills"]):
        assert O.seeded_fill(int(s), n, sc).tobytes() == arr[f"fill_{i}"].tobytes()


def test_buffer_axpy_golden(golden):
    arr, meta = golden
    y = np.array([1.0, 2.0, 3.0])
    O.buffer_axpy(2.0, np.array([10.0, 20.0, 30.0]), y)
    assert y.tolist() == arr["axpy_golden"].tolist() == [21.0, 42.0, 63.0]
    for i, a in enumerate(meta["axpy_alphas"]):
        y = arr["axpy_y0"].copy()
        O.buffer_axpy(a, arr["axpy_x"], y)
        assert y.tobytes() == arr[f"axpy_out_{i}"].tobytes()
    y32 = arr["axpy_y0"].astype(np.float32)
    O.buffer_axpy(1.0, arr["axpy_x"].astype(np.float32), y32)
    assert y32.tobytes() == arr["axpy32_out"].tobytes()


def test_master_update_golden(golden):
    arr, meta = golden
    out = O.master_update(np.array([1.0, 0.0, -1.0]), np.array([0.2, 0.0, -0.2]), 0.5)
    assert out.tolist() == [0.9, 0.0, -0.9] == arr["update_golden"].tolist()
    for i, eps in enumerate(meta["upd_eps"]):
        assert O.master_update(arr["upd_w"], arr["upd_g"], eps).tobytes() == arr[f"upd_out_{i}"].tobytes()
    got = O.master_update(arr["upd_w"].astype(np.float32), arr["upd_g"].astype(np.float32), 0.05)
    assert got.dtype == np.float64 and got.tobytes() == arr["upd32_out"].tobytes()
    assert np.array_equal(O.master_update_ref32(arr["upd_w"].astype(np.float32),
                                                arr["upd_g"].astype(np.float32), 0.05),
                          arr["upd32_out"].astype(np.float32))


def test_tree_shapes(golden):
    _, meta = golden
    for s in range(1, 17):
        parents = {int(k): v for k, v in meta["parents"][str(s)].items()}
        assert parents == {r: O.tree_parent(r) for r in range(1, s)}
        kids = {int(k): v for k, v in meta["children"][str(s)].items()}
        assert kids == {r: O.tree_children(r, s) for r in range(s)}
        assert O.tree_depth(s) == meta["depth"][str(s)]


@pytest.mark.parametrize("s", range(1, 9))
def test_tree_reduce_matches_reference(golden, s):
    arr, _ = golden
    parts = [[arr[f"tr{s}_in_{r}_0"], arr[f"tr{s}_in_{r}_1"]] for r in range(s)]
    out = O.tree_reduce(parts, s, np.float64)
    assert out[0].tobytes() == arr[f"tr{s}_out_0"].tobytes()
    assert out[1].tobytes() == arr[f"tr{s}_out_1"].tobytes()
    p32 = [[p[0].astype(np.float32)] for p in parts]
    assert O.tree_reduce(p32, s, np.float64)[0].tobytes() == arr[f"tr{s}_out32_0"].tobytes()
    assert O.tree_reduce(p32, s, np.float32)[0].tobytes() == arr[f"tr{s}_ref32_0"].tobytes()


def test_fold_order_under_cancellation(golden):
    arr, _ = golden
    parts = [[np.full(4, 1e16)], [np.full(4, 1.0)], [np.full(4, -1e16)], [np.full(4, 0.0)]]
    out = O.tree_reduce(parts, 4)[0]
    assert out.tolist() == [0.0] * 4 == arr["fold_1e16_out"].tolist()


def test_layout_rules(golden):
    _, meta = golden
    for e in meta["layouts"]:
        lay = O.Layout(e["counts"], e["chunk"])
        assert lay.layer_bytes == e["layer_bytes"]
        assert [int(x) for x in lay.layer_offsets] == e["layer_offsets"]
        assert lay.layer_chunks == e["layer_chunks"] and lay.bulk_chunks == e["bulk_chunks"]
        assert lay.model_notif_count() == e["model_notif_count"]
        assert lay.grad_notif_count(3) == e["grad_notif_count_3"]
        for l in range(lay.L):
            for p in (0, 1):
                assert lay.model_notif_base(l, p) == e["model_notif_base"][l][p]
                assert lay.model_slot_offset(l, p) == e["model_slot_offset"][l][p]
                for c in range(3):
                    assert lay.grad_notif_base(c, l, p) == e["grad_notif_base"][c][l][p]
                    assert lay.grad_slot_offset(c, l, p) == e["grad_slot_offset"][c][l][p]
        assert [lay.chunk_id(17, j, 5) for j in range(5)] == e["chunk_ids"]


def test_batches_and_shards(golden):
    _, meta = golden
    assert O.batch_indices(42, 7, 64, 100).tolist() == meta["batch_indices"]["42_7_64_100"]
    assert O.batch_indices(19, 3, 24, 48).tolist() == meta["batch_indices"]["19_3_24_48"]
    for w, spans in meta["shards"].items():
        assert [list(O.shard_bounds(64, int(w), r)) for r in range(int(w))] == spans


@pytest.mark.parametrize("ws", [1, 2, 3, 4, 8])
def test_e2e_replay_reproduces_reference_model(golden, ws):
    """Feeding the reference's per-rank gradients through the oracle exchange
    reproduces the reference engine's final model bit for bit."""
    arr, meta = golden
    e = [x for x in meta["e2e"] if x["world_size"] == ws][0]
    L = len(e["layers"])
    w = [arr[f"e2e{ws}_k0_w{l}"] for l in range(L)]
    for k in range(e["iterations"]):
        for l in range(L):
            assert w[l].tobytes() == arr[f"e2e{ws}_k{k}_w{l}"].tobytes()
            grads = [arr[f"e2e{ws}_k{k}_r{r}_l{l}"] for r in range(ws)]
            w[l] = O.exchange_iteration(grads, w[l], e["epsilon"], "ref64")
    for l in range(L):
        assert w[l].tobytes() == arr[f"e2e{ws}_final_l{l}"].tobytes()
    assert [sum(fc[l] for fc in e["fold_counts"]) for l in range(L)] == [(ws - 1) * e["iterations"]] * L
    assert e["barrier_calls"] == [0] * ws


def test_fast32_rule_is_caffe_order():
    """fast32 (parity unpinned vs the reference): check the restated Caffe order by hand."""
    w = np.array([1.0, -2.0], np.float32)
    v = np.array([0.5, 0.0], np.float32)
    g = np.array([0.25, 4.0], np.float32)
    w1, v1 = O.fast32_update(w, v, g, 0.5, 0.1, 0.9, 0.01)
    f = np.float32
    gg = f(0.5) * g + f(0.01) * w
    vv = f(0.9) * v + f(0.1) * gg
    assert np.array_equal(v1, vv.astype(f)) and np.array_equal(w1, (w - vv).astype(f))
