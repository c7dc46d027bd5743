"""Generate golden vectors for the gradient-exchange path from the REFERENCE itself.

Run in the build container only (it imports the read-only reference package):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written here is produced by calling the reference's own functions
(`pipesgd.buffers`, `pipesgd.topology`, `pipesgd.engine.sgd`, `pipesgd.engine.layout`,
`pipesgd.harness.run_inproc`).  The outputs are committed as `golden.npz` /
`golden.json` next to this script; tests and the oracle read only those files, so
nothing on the GPU box needs `/root/reference`.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from pipesgd import net  # noqa: E402
from pipesgd.buffers import buffer_axpy, derived_seed, mix64, seeded_fill, splitmix64_stream  # noqa: E402
from pipesgd.engine import SegmentLayout, TrainConfig, batch_indices, master_update, sequential_sgd, tree_reduce  # noqa: E402
from pipesgd.engine.sgd import shard_bounds  # noqa: E402
from pipesgd.harness import run_inproc  # noqa: E402
from pipesgd.topology import build_reduction_tree, depth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MASK = (1 << 64) - 1


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"source": "pipesgd 0.1.0 at /root/reference/pkg/src (reference package itself)"}

    # --- PRNG (buffers.py:23-66) ------------------------------------------------
    seeds = [0, 1, 42, 0xDEADBEEF, MASK]
    meta["splitmix_seeds"] = [str(s) for s in seeds]
    for i, s in enumerate(seeds):
        arrays[f"splitmix_{i}"] = splitmix64_stream(s, 17)
    meta["mix64"] = {str(z): str(mix64(z)) for z in (0, 1, 0x123456789ABCDEF0, MASK)}
    meta["derived_seed"] = [
        [42, [0, 3], str(derived_seed(42, 0, 3))],
        [42, [1, 0], str(derived_seed(42, 1, 0))],
        [7, [1, 2], str(derived_seed(7, 1, 2))],
        [MASK, [5], str(derived_seed(MASK, 5))],
    ]
    fills = [(9, 64, 0.5), (42 ^ 5, 4099, 1.0 / np.sqrt(9216.0)), (derived_seed(42, 1, 2), 1000, 1e-3)]
    meta["fills"] = [[str(s), n, sc] for s, n, sc in fills]
    for i, (s, n, sc) in enumerate(fills):
        arrays[f"fill_{i}"] = seeded_fill(s, n, sc)

    # --- buffer_axpy (buffers.py:69-74) -----------------------------------------
    y = np.array([1.0, 2.0, 3.0])
    buffer_axpy(2.0, np.array([10.0, 20.0, 30.0]), y)
    arrays["axpy_golden"] = y
    rng = np.random.default_rng(1234)
    ax_x = rng.normal(size=257) * 1e3
    ax_y = rng.normal(size=257)
    arrays["axpy_x"], arrays["axpy_y0"] = ax_x, ax_y.copy()
    for alpha_i, alpha in enumerate([1.0, -0.37, 3.0e-3]):
        out = ax_y.copy()
        buffer_axpy(alpha, ax_x, out)
        arrays[f"axpy_out_{alpha_i}"] = out
    meta["axpy_alphas"] = [1.0, -0.37, 3.0e-3]
    # fp32 arrays stay fp32 inside buffer_axpy (numpy in-place on float32)
    x32 = ax_x.astype(np.float32)
    y32 = ax_y.astype(np.float32)
    out32 = y32.copy()
    buffer_axpy(1.0, x32, out32)
    arrays["axpy32_out"] = out32

    # --- master_update (sgd.py:27-33) -------------------------------------------
    arrays["update_golden"] = master_update(np.array([1.0, 0.0, -1.0]), np.array([0.2, 0.0, -0.2]), 0.5)
    w = rng.normal(size=1001)
    g = rng.normal(size=1001) * 1e-2
    arrays["upd_w"], arrays["upd_g"] = w, g
    for i, eps in enumerate([0.05, 0.01, 0.3333333333333333]):
        arrays[f"upd_out_{i}"] = master_update(w, g, eps)
    meta["upd_eps"] = [0.05, 0.01, 0.3333333333333333]
    w32 = w.astype(np.float32)
    g32 = g.astype(np.float32)
    arrays["upd32_out"] = master_update(w32, g32, 0.05)  # f64 result (promotion inside)

    # --- trees (topology.py:34-55) -----------------------------------------------
    meta["parents"] = {}
    meta["children"] = {}
    meta["depth"] = {}
    for s in range(1, 17):
        t = build_reduction_tree(s)
        meta["parents"][s] = {str(k): v for k, v in t.parent.items()}
        meta["children"][s] = {str(k): v for k, v in t.children.items()}
        meta["depth"][s] = depth(t)

    # --- tree_reduce (sgd.py:53-69), f64 and fp32 inputs --------------------------
    for s in range(1, 9):
        parts = [[rng.normal(size=33) * (10.0 ** rng.integers(-3, 4)), rng.normal(size=5)] for _ in range(s)]
        for r in range(s):
            arrays[f"tr{s}_in_{r}_0"] = parts[r][0]
            arrays[f"tr{s}_in_{r}_1"] = parts[r][1]
        out = tree_reduce(parts, build_reduction_tree(s))
        arrays[f"tr{s}_out_0"], arrays[f"tr{s}_out_1"] = out[0], out[1]
        # fp32 partials: tree_reduce promotes to float64 (sgd.py:64)
        p32 = [[np.asarray(v, dtype=np.float32) for v in pr] for pr in parts]
        out32 = tree_reduce(p32, build_reduction_tree(s))
        arrays[f"tr{s}_out32_0"] = out32[0]
        # ref32 convention: the reference's buffer_axpy applied to fp32 arrays in tree order
        acc = [[np.array(v, dtype=np.float32, copy=True) for v in pr] for pr in p32]
        t = build_reduction_tree(s)
        for r in range(s - 1, -1, -1):
            for c in t.children[r]:
                buffer_axpy(1.0, acc[c][0], acc[r][0])
        arrays[f"tr{s}_ref32_0"] = acc[0][0]
    # the late-arrival fold-order case (test_turns.py:119-145): 1e16, 1.0, -1e16, 0
    parts = [[np.full(4, 1e16)], [np.full(4, 1.0)], [np.full(4, -1e16)], [np.full(4, 0.0)]]
    arrays["fold_1e16_out"] = tree_reduce(parts, build_reduction_tree(4))[0]

    # --- layout (layout.py:42-139) ------------------------------------------------
    lays = []
    for counts, chunk in [([10, 4, 6], 64), ([100, 1, 50], 64), ([3], 8), ([431080 // 4] * 4, 65536),
                          ([520, 25050, 400500, 5010], 65536)]:
        lay = SegmentLayout(counts, chunk)
        nc = 3
        entry = {
            "counts": counts, "chunk": chunk,
            "layer_bytes": lay.layer_bytes, "layer_offsets": lay.layer_offsets,
            "total_bytes": lay.total_bytes, "layer_chunks": lay.layer_chunks,
            "max_chunks": lay.max_chunks, "bulk_chunks": lay.bulk_chunks,
            "work_size": lay.work_size, "model_rx_size": lay.model_rx_size,
            "grad_rx_size_3": lay.grad_rx_size(nc), "grad_rx_size_0": lay.grad_rx_size(0),
            "model_notif_count": lay.model_notif_count, "grad_notif_count_3": lay.grad_notif_count(nc),
            "model_notif_base": [[lay.model_notif_base(l, p) for p in (0, 1)] for l in range(lay.num_layers)],
            "grad_notif_base": [[[lay.grad_notif_base(c, l, p) for p in (0, 1)] for l in range(lay.num_layers)]
                                for c in range(nc)],
            "model_bulk_base": [lay.model_bulk_base(p) for p in (0, 1)],
            "grad_bulk_base": [[lay.grad_bulk_base(nc, c, p) for p in (0, 1)] for c in range(nc)],
            "model_slot_offset": [[lay.model_slot_offset(l, p) for p in (0, 1)] for l in range(lay.num_layers)],
            "grad_slot_offset": [[[lay.grad_slot_offset(c, l, p) for p in (0, 1)] for l in range(lay.num_layers)]
                                 for c in range(nc)],
            "chunk_ids": [lay.chunk_notification_id(17, j, 5) for j in range(5)],
        }
        lays.append(entry)
    meta["layouts"] = lays

    # --- batch indices / shards (sgd.py:36-50) ----------------------------------
    meta["batch_indices"] = {
        "42_7_64_100": batch_indices(42, 7, 64, 100).tolist(),
        "19_3_24_48": batch_indices(19, 3, 24, 48).tolist(),
    }
    meta["shards"] = {str(w): [list(shard_bounds(64, w, r)) for r in range(w)] for w in (1, 2, 4, 8)}

    # --- end-to-end: reference engine vs oracle (test_equivalence.py:16-42) -------
    # A small MLP run; we store the per-iteration per-rank shard gradients the
    # reference produced, plus its final model, so the device exchange can be fed
    # exactly the reference's inputs and compared bit for bit.
    e2e = []
    for ws in (1, 2, 3, 4, 8):
        batch = 24
        cfg = TrainConfig(layer_dims=(6, 9, 5), world_size=ws, iterations=4, batch_size=batch,
                          dataset_size=48, seed=19, epsilon=0.08)
        ds = net.make_synthetic_dataset(cfg.seed, cfg.dataset_size, cfg.specs(), cfg.input_scale)
        specs = cfg.specs()
        model = net.init_model(cfg.seed, specs)
        tree = build_reduction_tree(ws)
        for k in range(cfg.iterations):
            idx = batch_indices(cfg.seed, k, cfg.batch_size, len(ds))
            for r in range(ws):
                lo, hi = shard_bounds(cfg.batch_size, ws, r)
                x, t = ds.take(idx[lo:hi])
                grads, _ = net.backward(specs, model.layers, x, t)
                for l, gl in enumerate(grads):
                    arrays[f"e2e{ws}_k{k}_r{r}_l{l}"] = gl
            for l in range(len(specs)):
                arrays[f"e2e{ws}_k{k}_w{l}"] = model.layers[l]
            partial = [[arrays[f"e2e{ws}_k{k}_r{r}_l{l}"] for l in range(len(specs))] for r in range(ws)]
            red = tree_reduce(partial, tree)
            from pipesgd.buffers import Model
            model = Model([master_update(model.layers[l], red[l], cfg.epsilon) for l in range(len(specs))], k + 1)
        ref = sequential_sgd(cfg, ds)
        for l in range(len(specs)):
            assert model.layers[l].tobytes() == ref.layers[l].tobytes()
            arrays[f"e2e{ws}_final_l{l}"] = ref.layers[l]
        results = run_inproc(cfg, ds)
        for res in results:
            for l in range(len(specs)):
                assert res.model[l].tobytes() == ref.layers[l].tobytes()
        e2e.append({"world_size": ws, "layers": [s.param_count for s in specs], "iterations": cfg.iterations,
                    "epsilon": cfg.epsilon, "fold_counts": [r.fold_counts for r in results],
                    "barrier_calls": [r.barrier_calls for r in results]})
    meta["e2e"] = e2e

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {os.path.getsize(os.path.join(OUT, 'golden.npz'))} bytes")


if __name__ == "__main__":
    main()
