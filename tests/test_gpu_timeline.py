"""The device timeline bench.py records, checked on the GPU.

bench.trace_timeline records, per traced step, a forward span, one backward_layer span per
layer (output-grad ready -> parameter grads final, the exchange trigger of
pipelined.py:91-95) and one send_trigger span per layer exchange, in the reference's CSV
schema (timeline.py:34).  This test runs it through the real hooks on cuda:0 (LeNet, one
rank: the exchange is the fused update) and checks

* the CSV round-trips through the reference-compatible reader (timeline.py:56-110);
* the overlap ratio equals the oracle's restatement of timeline.py:137-175 on the same
  events, and the package's compute_overlap;
* the spans are well formed: every layer has one backward_layer and one send_trigger span
  per step, layers finish backward in decreasing order, and each layer's exchange starts
  exactly when its backward span ends (gradient-ready event).
"""

import types

import numpy as np
import pytest
import torch

from oracle import pipesgd_oracle as O

pytestmark = pytest.mark.gpu


def test_device_timeline_matches_oracle_metrics(cuda, tmp_path):
    import bench
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.timeline import compute_overlap, read_timeline_csv
    from paper_1706_00095_b200.transport import LocalWorld
    from workloads import WORKLOADS

    wl = WORKLOADS["lenet"]
    dev = torch.device("cuda", 0)
    model = wl["cls"]().to(dev)
    sizes = [sum(p.numel() for p in ps) for _, ps in model.layers()]
    world = LocalWorld(1, inline=False)
    tr = world.transport(0)
    xchg = DeviceExchange(tr, sizes, mode="fast32", variant="auto", chunk_elems=16384, scale=1.0, **wl["hyper"])
    bind = ModuleBinding(xchg, model.layers(), gate="layer")
    xchg.connect()
    g = torch.Generator().manual_seed(0)
    B, C, IMG = bench.global_batch(wl, 1), wl.get("channels", 3), wl["image"]
    dev_x = torch.randint(0, 256, (B, C, IMG, IMG), dtype=torch.uint8, generator=g).to(dev)
    dev_y = torch.randint(0, wl.get("classes", 1000), (B,), dtype=torch.int64, generator=g).to(dev)
    path = str(tmp_path / "timeline_rank{rank}.csv")
    args = types.SimpleNamespace(timeline=path)
    steps = 3
    out = bench.trace_timeline(args, bind, model, None, dev_x, dev_y, 0, 1, steps=steps)
    torch.cuda.synchronize()

    ev = read_timeline_csv(path.replace("{rank}", "0"))
    L = len(sizes)
    assert out["backward_layer_spans"] == steps * L
    by = {}
    for e in ev:
        by.setdefault((e.kind, e.iteration, e.layer), []).append(e)
    its = sorted({e.iteration for e in ev})
    assert len(its) == steps
    for k in its:
        assert len(by[("forward", k, -1)]) == 1
        ends = []
        for l in range(L):
            (b,) = by[("backward_layer", k, l)]
            (s,) = by[("send_trigger", k, l)]
            assert b.t_start_ns <= b.t_end_ns and s.t_start_ns <= s.t_end_ns
            assert s.t_start_ns == b.t_end_ns  # the exchange is triggered by the gradient-ready event
            ends.append(b.t_end_ns)
        assert ends == sorted(ends, reverse=True)  # emission order L-1 ... 0 (net.py:207-214)
    tuples = [(e.rank, e.iteration, e.layer, e.kind, e.t_start_ns, e.t_end_ns) for e in ev]
    want = O.overlap_metrics(tuples)
    got = compute_overlap(ev)
    assert got.overlap_ratio == want["overlap_ratio"] == out["overlap_ratio"]
    assert np.isfinite(got.overlap_ratio) and 0.0 <= got.overlap_ratio <= 1.0
    xchg.close()
    world.close()
