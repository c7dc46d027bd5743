"""Golden vectors for the data formats either side of the path,
produced by the REFERENCE itself: the PSGD1 checkpoint (engine/checkpoint.py) and the
timeline CSV / overlap metrics (timeline.py).

Run in the build container only (imports the read-only reference package):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_formats.py

Writes formats_golden.npz / formats_golden.json next to this script.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from pipesgd.buffers import seeded_fill  # noqa: E402
from pipesgd.engine.checkpoint import load_model_bytes, serialize_model  # noqa: E402
from pipesgd.errors import FormatError  # noqa: E402
from pipesgd.timeline import TimelineEvent, compute_overlap, read_timeline_csv  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
LENET = [520, 25050, 400500, 5010]


def small_layers():
    """Edge values: signed zeros, subnormals, inf/nan, extremes, plus seeded data."""
    special = np.array([0.0, -0.0, 1.0, -1.0, 5e-324, -2.2250738585072014e-308, np.inf, -np.inf, np.nan,
                        1.7976931348623157e308, 0.1, 1 / 3], dtype=np.float64)
    return [special, seeded_fill(7, 1, 1.0), seeded_fill(8, 17, 1e-3), seeded_fill(9, 300, 2.5)]


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"source": "pipesgd at /root/reference/pkg/src (engine/checkpoint.py, timeline.py)"}

    # ---- PSGD1 checkpoints
    layers = small_layers()
    blob = serialize_model(layers)
    arrays["ckpt_small_blob"] = np.frombuffer(blob, dtype=np.uint8).copy()
    for i, a in enumerate(layers):
        arrays[f"ckpt_small_l{i}"] = a
    # fp32 weights as the exchange holds them: the reference serializes their f64 promotion
    lenet32 = [seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)).astype(np.float32) for l, n in enumerate(LENET)]
    blob32 = serialize_model(lenet32)
    meta["ckpt_lenet_f32_sha256"] = hashlib.sha256(blob32).hexdigest()
    meta["ckpt_lenet_f32_bytes"] = len(blob32)
    lenet64 = [seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)) for l, n in enumerate(LENET)]
    blob64 = serialize_model(lenet64)
    meta["ckpt_lenet_f64_sha256"] = hashlib.sha256(blob64).hexdigest()
    back = load_model_bytes(blob64)
    assert all(np.array_equal(a, b) for a, b in zip(back.layers, lenet64))

    bad = {
        "magic": b"PSGD2" + blob[5:],
        "empty": b"PSGD1",
        "partial_header": blob[:5 + 7],
        "short_layer": blob[:5 + 12 + 8 * 5],
        "index": blob[:5] + (1).to_bytes(4, "little") + blob[9:],
    }
    meta["ckpt_errors"] = {}
    for k, b in bad.items():
        try:
            load_model_bytes(b)
            meta["ckpt_errors"][k] = None
        except FormatError as exc:
            meta["ckpt_errors"][k] = str(exc)
        arrays[f"ckpt_bad_{k}"] = np.frombuffer(b, dtype=np.uint8).copy()

    # ---- timeline overlap on seeded random event sets
    rng = np.random.default_rng(1706)
    kinds = ["forward", "backward_layer", "reduce_local", "send_trigger", "recv_notify", "master_update",
             "model_forward", "finalize", "barrier"]
    cases = []
    for c in range(6):
        evs = []
        for _ in range(int(rng.integers(0, 40))):
            t0 = int(rng.integers(0, 10_000))
            evs.append(TimelineEvent(int(rng.integers(0, 3)), int(rng.integers(0, 4)), int(rng.integers(-1, 5)),
                                     kinds[int(rng.integers(0, len(kinds)))], t0, t0 + int(rng.integers(0, 3000))))
        m = compute_overlap(evs)
        cases.append({"events": [[e.rank, e.iteration, e.layer, e.kind, e.t_start_ns, e.t_end_ns] for e in evs],
                      "overlap_ratio": m.overlap_ratio, "iterations_per_second": m.iterations_per_second,
                      "wall_clock_ns": {str(k): v for k, v in m.wall_clock_ns.items()},
                      "per_rank_overlap": {str(k): v for k, v in m.per_rank_overlap.items()},
                      "lines": m.lines()})
    meta["overlap_cases"] = cases

    # ---- timeline CSV reader errors (the message after the path prefix)
    header = "rank,iteration,layer,kind,t_start_ns,t_end_ns\n"
    csvs = {
        "header": "rank,iter,layer,kind,t0,t1\n",
        "columns": header + "0,0,1,forward,5\n",
        "int": header + "0,0,x,forward,5,6\n",
        "kind": header + "0,0,1,fwd,5,6\n",
        "order": header + "0,0,1,forward,6,5\n",
        "ok_blank": header + "\n0,0,1,forward,5,6\n\n1,2,-1,barrier,0,0\n",
    }
    meta["csv_cases"] = {}
    with tempfile.TemporaryDirectory() as d:
        for k, text in csvs.items():
            p = os.path.join(d, "t.csv")
            with open(p, "w") as fh:
                fh.write(text)
            try:
                got = read_timeline_csv(p)
                res = {"events": [[e.rank, e.iteration, e.layer, e.kind, e.t_start_ns, e.t_end_ns] for e in got]}
            except FormatError as exc:
                res = {"error": str(exc).replace(p, "{path}")}
            meta["csv_cases"][k] = {"text": text, **res}

    np.savez_compressed(os.path.join(OUT, "formats_golden.npz"), **arrays)
    with open(os.path.join(OUT, "formats_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays,", len(meta), "meta keys")


if __name__ == "__main__":
    main()
