"""The exchange configuration bench.py runs, compared bit for bit with the oracle.

bench.py builds `DeviceExchange(variant="auto", chunk_elems=16384, scale=1/N, large="ce",
flags=("allow_l128",), l128_range=L128_BAND)` over the AlexNet layer list (and GoogLeNet's
64 layers with the whole-model gate).  At N >= 2 that sends fc6/fc7/fc8 to the copy-engine
two-shot with its owner shard split into pipelined parts (`ce_split`), conv2-5 to the
128-byte-line two-shot (TWOSHOT_L128), and conv1 to the LL one-shot.  These tests drive exactly that plan, ranks
emulated on ONE GPU with every phase launched in dependency order (test_gpu_exchange's
single-GPU hazard rule), and require the weights every rank holds to equal the
oracle's tree-order fold + update (pipelined.py:158-203, sgd.py:27-33; the bar is the
reference's bit-identical grids, tests/test_equivalence.py:36-42).

Gradients are numpy PCG64 draws (seeded per rank/layer/iteration): the arithmetic under
test does not depend on how the inputs were made, and drawing 8 x 61 M values with
`seeded_fill` would dominate the run.  Comparisons are bitwise on the device.
"""

import numpy as np
import pytest
import torch

from oracle import pipesgd_oracle as O

from test_gpu_exchange import build, stepped_layer

pytestmark = pytest.mark.gpu

ALEXNET = [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]  # bench.py / SURVEY §8
HYPER = dict(lr=0.01, momentum=0.9, weight_decay=5e-4)  # workloads.WORKLOADS["alexnet"]["hyper"]


def _googlenet_sizes():
    from workloads import GoogLeNet

    return [sum(p.numel() for p in ps) for _, ps in GoogLeNet().layers()]


def _grad(r, l, k, n):
    rng = np.random.default_rng([r, l, k, 7])
    return (rng.standard_normal(n, dtype=np.float32) * np.float32(1e-2)).astype(np.float32)


def _bits_equal(t, a):
    want = torch.from_numpy(np.ascontiguousarray(a)).to(t.device)
    return torch.equal(t.view(torch.int32), want.view(torch.int32))


def _expected_variants(sizes, N, mode, large="ce"):
    from paper_1706_00095_b200.exchange import L128_BAND, choose_variant

    ll = (1 << 16) if mode != "ref64" else 0
    band = L128_BAND if mode != "ref64" else (0, 0)
    return [choose_variant(n, N, 0, ce_from=1 << 20, large=large, ll_below=ll, l128_range=band) for n in sizes]


def _run(N, sizes, mode, iters, gate, fast_hyper=HYPER, large="ce", overlap_ctas=16, flags=()):
    from paper_1706_00095_b200.exchange import L128_BAND

    hyper = fast_hyper if mode == "fast32" else dict(lr=0.05)
    # bench.py's defaults: --l128 = L128_BAND (with the allow_l128 opt-in), large layers "ce",
    # --overlap-ctas 16
    world, trs, xs = build(N, sizes, mode, "auto", chunk_elems=16384, flags=("allow_l128",) + tuple(flags),
                           l128_range=L128_BAND,
                           large=large, overlap_ctas=overlap_ctas, **hyper)
    if overlap_ctas:  # every small layer but layer 0 runs on the capped grid
        caps = [xs[0].layer_plan(l)[1] for l in range(len(sizes))]
        assert all(c <= overlap_ctas for l, c in enumerate(caps) if l > 0 and sizes[l] < (1 << 20)), caps
    assert xs[0].variants == _expected_variants(sizes, N, mode, large)
    w = [O.seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)).astype(np.float32) for l, n in enumerate(sizes)]
    v = [np.zeros(n, np.float32) for n in sizes]
    for x in xs:
        for l in range(len(sizes)):
            x.layer_views[l].copy_(torch.from_numpy(w[l]))
    torch.cuda.synchronize()
    for k in range(iters):
        for l in reversed(range(len(sizes))):  # backward emission order
            n = sizes[l]
            grads = [_grad(r, l, k, n) for r in range(N)]
            # [dW][db] pieces as autograd hands them over (bias = the last <= 4096 values)
            cut = n - min(4096, max(1, n // 64))
            pieces = [[torch.from_numpy(g[:cut]).cuda(), torch.from_numpy(g[cut:]).cuda()] for g in grads]
            stepped_layer(xs, trs, l, k, pieces, gate=(gate == "layer"))
            if mode == "fast32":
                w[l], v[l] = O.exchange_iteration(grads, w[l], hyper["lr"], mode, state=v[l], scale=1.0 / N,
                                                  momentum=hyper["momentum"], weight_decay=hyper["weight_decay"])
            else:
                w[l] = O.exchange_iteration(grads, w[l], 0.05, mode).astype(np.float32)
            del pieces, grads
        if gate == "model":  # one whole-model gate per rank (ModuleBinding gate="model")
            for r in range(N):
                xs[r].gate_all(k, stream=trs[r].stream)
            torch.cuda.synchronize()
        for l in range(len(sizes)):
            for r in range(N):
                assert _bits_equal(xs[r].layer_views[l], w[l]), \
                    f"N={N} {mode} iteration {k} layer {l} ({sizes[l]} params, {xs[0].variants[l]}) rank {r}"
    for tr in trs:
        assert tr.device_status() == 0
    for x in xs:
        x.close()
    world.close()


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("mode", ["fast32", "ref32"])
@pytest.mark.parametrize("large", ["ce", "cet", "bulk"])
def test_alexnet_auto_plan_matches_oracle(cuda, N, mode, large):
    """The AlexNet step's exchange plan (copy-engine two-shot with 3-4 owner parts for
    fc6/fc7/fc8, auto-sized chunks elsewhere), two iterations, every rank bit-exact; also
    with bench.py's --large cet (TMA-fed owner fold) and --large bulk (TMA bulk kernel)."""
    _run(N, ALEXNET, mode, iters=2, gate="layer", large=large)


def test_alexnet_plan_has_multipart_owners(cuda):
    """Guard: the copy-engine layers really run with several pipelined owner parts, the
    path these parity tests exist for (ce_split, pgx_xchg.cu)."""
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import LocalWorld

    for N in (2, 4, 8):
        world = LocalWorld(N, inline=False)
        tr = [world.transport(r) for r in range(N)]
        x = DeviceExchange(tr[0], ALEXNET, mode="fast32", variant="auto", chunk_elems=16384, **HYPER)
        parts = [x.ce_parts(l) for l in range(len(ALEXNET))]
        assert parts[5] >= 3 and parts[6] >= 3, (N, parts)  # fc6, fc7
        x.close()
        world.close()


@pytest.mark.parametrize("N", [4, 8])
@pytest.mark.parametrize("overlap_ctas,lean", [(0, False), (16, False), (16, True)])
def test_googlenet_auto_plan_model_gate_matches_oracle(cuda, N, overlap_ctas, lean):
    """GoogLeNet's 64 layers (12 KB .. 8 MB) with the whole-model gate bench.py uses for
    nets of > 16 layers: LL / one-shot / two-shot / copy-engine layers in one step; also
    with the hidden small layers on 16-CTA grids (bench.py --overlap-ctas)."""
    _run(N, _googlenet_sizes(), "fast32", iters=2, gate="model", overlap_ctas=overlap_ctas,
         flags=("lean_capped",) if lean else ())


@pytest.mark.parametrize("workload,N", [("lenet", 2), ("cifar10_quick", 4)])
def test_small_net_auto_plans_match_oracle(cuda, workload, N):
    """BASELINE configs[0] (LeNet-5, 2 ranks) and configs[1] (cifar10_quick, 4 ranks) with
    their own SGD hyper-parameters (workloads.WORKLOADS), the plan bench.py runs for them."""
    from workloads import WORKLOADS

    wl = WORKLOADS[workload]
    sizes = [sum(p.numel() for p in ps) for _, ps in wl["cls"]().layers()]
    _run(N, sizes, "fast32", iters=3, gate="layer", fast_hyper=wl["hyper"])
