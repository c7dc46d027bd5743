"""Device-driven exchange (two-shot and the paper's tree) vs the CPU oracle.

Ranks are emulated on ONE GPU by launching each phase of every rank in dependency
order with a synchronize in between, so no kernel ever spins on a kernel that has
not been launched (single-GPU hazard rule); the real concurrent multi-GPU path is
in test_gpu_multi.py.
"""

import numpy as np
import pytest
import torch

from oracle import pipesgd_oracle as O

pytestmark = pytest.mark.gpu

LENET = [520, 25050, 400500, 5010]
CIFAR = [2432, 25632, 51264, 65600, 650]


def build(N, elems, mode, variant, chunk_elems=4096, **kw):
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import LocalWorld

    world = LocalWorld(N, inline=False)
    trs = [world.transport(r) for r in range(N)]
    if variant in ("oneshot_l128", "twoshot_l128"):  # opt-in only (pgx.h PGX_XF_ALLOW_L128)
        kw.setdefault("flags", ("allow_l128",))
    xs = [DeviceExchange(tr, elems, mode=mode, variant=variant, chunk_elems=chunk_elems, **kw) for tr in trs]
    for x in xs:
        x.connect()
    return world, trs, xs


def stepped_layer(xs, trs, l, k, pieces_by_rank, gate=True):
    from paper_1706_00095_b200 import _lib

    N = len(xs)
    sync = torch.cuda.synchronize
    if xs[0].variants[l] in ("twoshot", "twoshot_ce", "twoshot_cep", "oneshot", "oneshot_ll", "oneshot_l128",
                            "twoshot_bulk", "twoshot_ceb", "twoshot_cet"):
        for r in range(N):
            xs[r].launch(l, k, pieces_by_rank[r], stream=trs[r].stream, phases=_lib.PHASE_PUSH)
        sync()
        for r in range(N):
            xs[r].launch(l, k, pieces_by_rank[r], stream=trs[r].stream, phases=_lib.PHASE_OWNER)
            sync()
    elif xs[0].variants[l] == "twoshot_l128":  # push, owner (fold + update + gather), install
        for ph in (_lib.PHASE_PUSH, _lib.PHASE_OWNER, _lib.PHASE_DOWN):
            for r in range(N):
                xs[r].launch(l, k, pieces_by_rank[r], stream=trs[r].stream, phases=ph)
            sync()
    else:
        for r in reversed(range(N)):  # children (higher ranks) before parents
            xs[r].launch(l, k, pieces_by_rank[r], stream=trs[r].stream, phases=_lib.PHASE_PUSH)
            sync()
        for r in range(N):  # parents before children
            xs[r].launch(l, k, pieces_by_rank[r], stream=trs[r].stream, phases=_lib.PHASE_DOWN)
            sync()
    if gate:
        for r in range(N):
            xs[r].gate(l, k, stream=trs[r].stream)
    sync()
    for tr in trs:
        assert tr.device_status() == 0


def split_pieces(g, cut):
    if cut is None or cut <= 0 or cut >= g.numel():
        return [g]
    return [g[:cut].contiguous(), g[cut:].contiguous()]


@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("variant", ["twoshot", "tree", "twoshot_ce", "twoshot_cep", "oneshot", "oneshot_ll",
                                     "oneshot_l128", "twoshot_bulk", "twoshot_l128", "twoshot_ceb", "twoshot_cet"])
@pytest.mark.parametrize("mode", ["ref32", "fast32", "ref64", "sum32"])
def test_exchange_matches_oracle(cuda, N, variant, mode):
    if variant in ("oneshot_ll", "oneshot_l128", "twoshot_l128") and mode == "ref64":
        pytest.skip("the LL one-shots carry fp32 values")
    elems = LENET if N in (2, 8) else CIFAR
    iters = 3
    dt = np.float64 if mode == "ref64" else np.float32
    tdt = torch.float64 if mode == "ref64" else torch.float32
    hyper = dict(lr=0.01, momentum=0.9, weight_decay=5e-4) if mode == "fast32" else dict(lr=0.05)
    world, trs, xs = build(N, elems, mode, variant, **hyper)
    w = [O.seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)).astype(dt) for l, n in enumerate(elems)]
    v = [np.zeros(n, np.float32) for n in elems]
    for x in xs:
        for l in range(len(elems)):
            x.layer_views[l].copy_(torch.from_numpy(w[l]))
    torch.cuda.synchronize()
    for k in range(iters):
        for l in reversed(range(len(elems))):  # backward emission order
            n = elems[l]
            grads = [O.seeded_fill(O.derived_seed(42, r, l, k), n, 1e-2).astype(dt) for r in range(N)]
            cut = n - 4 if l % 2 == 0 else n - 3  # [W][b]-style pieces, aligned and ragged cuts
            pieces = [split_pieces(torch.from_numpy(g).to("cuda", tdt), cut) for g in grads]
            stepped_layer(xs, trs, l, k, pieces)
            if mode == "fast32":
                w[l], v[l] = O.exchange_iteration(grads, w[l], 0.01, mode, state=v[l], scale=1.0 / N,
                                                  momentum=0.9, weight_decay=5e-4)
            elif mode == "sum32":  # update off: every rank holds the averaged tree-order sum
                w[l] = O.exchange_iteration(grads, w[l], 0.05, mode, scale=1.0 / N)
            else:
                w[l] = O.exchange_iteration(grads, w[l], 0.05, mode).astype(dt)
            for r in range(N):
                got = xs[r].layer_views[l].cpu().numpy()
                if mode == "fast32":
                    np.testing.assert_allclose(got, w[l], rtol=1e-5, atol=1e-7)
                assert got.tobytes() == w[l].tobytes(), f"rank {r} layer {l} iteration {k}"
    for x in xs:
        x.close()
    world.close()


def test_exchange_bytes_accounting(cuda):
    world, trs, xs = build(4, LENET, "fast32", "twoshot", lr=0.01)
    nvl, hbm = xs[0].layer_bytes(2)
    own = -(-(-(-400500 // 4)) // 4) * 4  # rank 0's shard: ceil(S/N) rounded up to 4 elements
    assert nvl == 2 * (400500 - own) * 4
    for x in xs:
        x.close()
    world.close()


def test_module_binding_single_gpu_matches_sgd_rule(cuda):
    """N=1: the hook-driven fused update equals the fast32 oracle on a real module."""
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import LocalWorld

    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.ReLU(), torch.nn.Flatten(),
                              torch.nn.Linear(8 * 6 * 6, 10)).cuda()
    mods = [net[0], net[3]]
    layers = [(m, [m.weight, m.bias]) for m in mods]
    elems = [sum(p.numel() for p in ps) for _, ps in layers]
    world = LocalWorld(1, inline=False)
    tr = world.transport(0)
    x = DeviceExchange(tr, elems, mode="fast32", lr=0.1, momentum=0.9, weight_decay=1e-3)
    x.connect()
    bind = ModuleBinding(x, layers)
    w = [torch.cat([p.detach().reshape(-1) for p in ps]).cpu().numpy() for _, ps in layers]
    v = [np.zeros_like(a) for a in w]
    data = torch.randn(4, 3, 8, 8, device="cuda")
    for k in range(3):
        loss = net(data).square().mean()
        loss.backward()
        bind.step_done()
        # oracle from the same gradients: recompute them on a detached copy
        bind.drain()
        torch.cuda.synchronize()
        got = [x.layer_views[l].cpu().numpy() for l in range(2)]
        # reproduce: gradients at the pre-update weights
        ref_net = torch.nn.Sequential(torch.nn.Conv2d(3, 8, 3), torch.nn.ReLU(), torch.nn.Flatten(),
                                      torch.nn.Linear(8 * 6 * 6, 10)).cuda()
        with torch.no_grad():
            for m, a in zip([ref_net[0], ref_net[3]], w):
                t = torch.from_numpy(a).cuda()
                m.weight.copy_(t[:m.weight.numel()].view_as(m.weight))
                m.bias.copy_(t[m.weight.numel():])
        ref_net(data).square().mean().backward()
        for l, m in enumerate([ref_net[0], ref_net[3]]):
            g = torch.cat([m.weight.grad.reshape(-1), m.bias.grad]).cpu().numpy()
            w[l], v[l] = O.fast32_update(w[l], v[l], g, 1.0, 0.1, 0.9, 1e-3)
            np.testing.assert_allclose(got[l], w[l], rtol=1e-5, atol=1e-6)
    bind.remove()
    x.close()
    world.close()


def test_module_binding_disabled_launches_nothing(cuda):
    """bench.py's fwd_bwd_alone: with the binding disabled a backward launches no exchange,
    gates nothing, leaves the weights untouched and drops the gradients; re-enabled, the
    next step exchanges as usual."""
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import LocalWorld

    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(16, 8), torch.nn.ReLU(), torch.nn.Linear(8, 4)).cuda()
    layers = [(m, [m.weight, m.bias]) for m in (net[0], net[2])]
    elems = [sum(p.numel() for p in ps) for _, ps in layers]
    world = LocalWorld(1, inline=False)
    x = DeviceExchange(world.transport(0), elems, mode="fast32", lr=0.1, momentum=0.9)
    x.connect()
    bind = ModuleBinding(x, layers)
    data = torch.randn(5, 16, device="cuda")
    before = x.model.clone()
    n0, l0 = x.launch_count(), bind.gpu_launches
    bind.disabled = True
    net(data).square().mean().backward()
    torch.cuda.synchronize()
    assert x.launch_count() == n0 and bind.gpu_launches == l0
    assert torch.equal(x.model, before)
    assert all(p.grad is None for _, ps in layers for p in ps)
    bind.disabled = False
    net(data).square().mean().backward()
    bind.step_done()
    bind.drain()
    torch.cuda.synchronize()
    assert bind.gpu_launches > l0 and not torch.equal(x.model, before)
    assert x.tr.device_status() == 0
    bind.remove()
    x.close()
    world.close()


class _FixedGrad(torch.nn.Module):
    """loss = sum(w * c) + sum(b * d): its gradient is exactly (c, d) every step (no GEMM
    rounding), so graph replays and eager steps must both equal the oracle bit for bit."""

    def __init__(self, n, seed):
        super().__init__()
        gen = torch.Generator().manual_seed(seed)
        self.weight = torch.nn.Parameter(torch.randn(n, generator=gen).cuda())
        self.bias = torch.nn.Parameter(torch.randn(7, generator=gen).cuda())
        self.c = (torch.randn(n, generator=gen) * 1e-2).cuda()
        self.d = (torch.randn(7, generator=gen) * 1e-2).cuda()

    def forward(self):
        return (self.weight * self.c).sum() + (self.bias * self.d).sum()


@pytest.mark.parametrize("variant", ["twoshot", "twoshot_ce", "twoshot_cep", "oneshot", "oneshot_ll", "twoshot_bulk",
                                     "twoshot_l128", "twoshot_ceb", "twoshot_cet"])
@pytest.mark.parametrize("gate", ["layer", "model"])
def test_cuda_graph_replay_matches_oracle(cuda, variant, gate):
    """A captured training step (device iteration counter) applies exactly the oracle update."""
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import LocalWorld

    m = _FixedGrad(40000, 5)
    layers = [(m, [m.weight, m.bias])]
    world = LocalWorld(1, inline=False)
    tr = world.transport(0)
    x = DeviceExchange(tr, [40007], mode="fast32", variant=variant, lr=0.05, momentum=0.9, weight_decay=1e-3,
                       flags=(("allow_l128",) if "l128" in variant else ()))
    x.connect()
    w = torch.cat([m.weight.detach(), m.bias.detach()]).cpu().numpy()
    g = torch.cat([m.c, m.d]).cpu().numpy()
    bind = ModuleBinding(x, layers, gate=gate)
    v = np.zeros_like(w)

    def step():
        m().backward()
        bind.step_done()

    for _ in range(2):
        step()
    bind.drain()
    torch.cuda.synchronize()
    x.set_device_iteration(True, bind.k - 1)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap), torch.cuda.graph(graph, stream=cap):
        bind.begin_step()
        step()
        bind.drain()
    torch.cuda.current_stream().wait_stream(cap)
    for _ in range(4):
        graph.replay()
    bind.wait_current()
    torch.cuda.synchronize()
    for _ in range(6):
        w, v = O.fast32_update(w, v, g, 1.0, 0.05, 0.9, 1e-3)
    assert tr.device_status() == 0
    assert x.layer_views[0].cpu().numpy().tobytes() == w.tobytes()
    bind.remove()
    x.close()
    world.close()


@pytest.mark.parametrize("variant", ["twoshot", "tree", "twoshot_ce", "twoshot_cep", "oneshot", "oneshot_ll",
                                     "oneshot_l128", "twoshot_bulk", "twoshot_l128", "twoshot_ceb", "twoshot_cet"])
def test_tiny_and_ragged_layers_at_eight_ranks(cuda, variant):
    """Layers smaller than one vector per rank (empty owner shards), ragged tails and a
    piece boundary inside a vector, 8 ranks stepped on one GPU, ref32 bit-exact."""
    elems = [1, 3, 5, 17, 33, 4097]
    N = 8
    world, trs, xs = build(N, elems, "ref32", variant, chunk_elems=8, lr=0.125)
    w = [O.seeded_fill(9 ^ l, n, 1.0).astype(np.float32) for l, n in enumerate(elems)]
    for x in xs:
        for l in range(len(elems)):
            x.layer_views[l].copy_(torch.from_numpy(w[l]))
    torch.cuda.synchronize()
    for k in range(2):
        for l in reversed(range(len(elems))):
            n = elems[l]
            grads = [O.seeded_fill(O.derived_seed(3, r, l, k), n, 1.0).astype(np.float32) for r in range(N)]
            pieces = [split_pieces(torch.from_numpy(g).cuda(), n // 2) for g in grads]
            stepped_layer(xs, trs, l, k, pieces)
            w[l] = O.exchange_iteration(grads, w[l], 0.125, "ref32")
            for r in range(N):
                assert xs[r].layer_views[l].cpu().numpy().tobytes() == w[l].tobytes(), (variant, k, l, r)
    for x in xs:
        x.close()
    world.close()


def test_size_scaled_chunks_and_parity(cuda):
    """Big shards get larger chunks (fewer system fences) — the result stays bit-exact."""
    N, n = 4, (1 << 24) + 12
    world, trs, xs = build(N, [n, 4096], "fast32", "twoshot", chunk_elems=16384, lr=0.01, momentum=0.9)
    assert xs[0].layer_plan(0)[0] == 32768  # shard ~4.2 M elements -> >= 128 chunks of 32 K
    assert xs[0].layer_plan(1)[0] == 8192  # small shard (<= 256 K elements): half chunks
    w = O.seeded_fill(7, n, 0.05).astype(np.float32)
    for x in xs:
        x.layer_views[0].copy_(torch.from_numpy(w))
    grads = [O.seeded_fill(O.derived_seed(1, r), n, 1e-2).astype(np.float32) for r in range(N)]
    stepped_layer(xs, trs, 0, 0, [[torch.from_numpy(g).cuda()] for g in grads])
    want, _ = O.exchange_iteration(grads, w, 0.01, "fast32", state=np.zeros(n, np.float32), scale=1.0 / N,
                                   momentum=0.9, weight_decay=0.0)
    for r in range(N):
        assert xs[r].layer_views[0].cpu().numpy().tobytes() == want.tobytes()
    for x in xs:
        x.close()
    world.close()


class _Chain(torch.nn.Module):
    """y = x + sum(w*c) + sum(b*d): chained in a model, every layer's gradient is exactly
    (c, d), and later layers' backward allocations would reuse freed gradient memory."""

    def __init__(self, n, seed):
        super().__init__()
        gen = torch.Generator().manual_seed(seed)
        self.weight = torch.nn.Parameter(torch.randn(n, generator=gen).cuda())
        self.bias = torch.nn.Parameter(torch.randn(7, generator=gen).cuda())
        self.c = (torch.randn(n, generator=gen) * 1e-2).cuda()
        self.d = (torch.randn(7, generator=gen) * 1e-2).cuda()

    def forward(self, x):
        return x + (self.weight * self.c).sum() + (self.bias * self.d).sum()


@pytest.mark.parametrize("gate", ["layer", "model"])
def test_cuda_graph_multi_layer_single_gpu(cuda, gate):
    """Several layers in one captured step on one GPU: each layer's fused update must read
    its own gradient, not memory a later layer's backward reused (graph-lifetime keep)."""
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import LocalWorld

    sizes = [3000, 70000, 400000, 1500000]
    mods = [_Chain(n, 11 + i) for i, n in enumerate(sizes)]
    layers = [(m, [m.weight, m.bias]) for m in mods]
    world = LocalWorld(1, inline=False)
    tr = world.transport(0)
    x = DeviceExchange(tr, [n + 7 for n in sizes], mode="fast32", variant="auto", lr=0.05, momentum=0.9,
                       weight_decay=1e-3)
    x.connect()
    bind = ModuleBinding(x, layers, gate=gate)
    w = [torch.cat([m.weight.detach(), m.bias.detach()]).cpu().numpy() for m in mods]
    g = [torch.cat([m.c, m.d]).cpu().numpy() for m in mods]
    v = [np.zeros_like(a) for a in w]

    def step():
        y = torch.zeros((), device="cuda")
        for m in mods:
            y = m(y)
        y.backward()
        bind.step_done()

    for _ in range(2):
        step()
    bind.drain()
    torch.cuda.synchronize()
    x.set_device_iteration(True, bind.k - 1)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap), torch.cuda.graph(graph, stream=cap):
        bind.begin_step()
        step()
        bind.drain()
    torch.cuda.current_stream().wait_stream(cap)
    for _ in range(3):
        graph.replay()
    bind.wait_current()
    torch.cuda.synchronize()
    for l in range(len(sizes)):
        for _ in range(5):  # 2 eager steps + 3 replays (capturing runs nothing)
            w[l], v[l] = O.fast32_update(w[l], v[l], g[l], 1.0, 0.05, 0.9, 1e-3)
        assert x.layer_views[l].cpu().numpy().tobytes() == w[l].tobytes(), f"layer {l}"
    assert tr.device_status() == 0
    bind.remove()
    x.close()
    world.close()


@pytest.mark.parametrize("N", [2, 3, 4, 8])
def test_ceb_part_major_reduce_scatter_matches_oracle(cuda, N):
    """TWOSHOT_BULK with the copy-engine reduce-scatter (twoshot_ceb): a layer with enough
    slabs per shard for every one of the part-major copies + per-part chunk signals, a ragged
    [W][b] piece cut inside a part, three iterations, fast32 bit-exact."""
    elems = [4099, 3_000_003]
    world, trs, xs = build(N, elems, "fast32", "twoshot_ceb", lr=0.01, momentum=0.9, weight_decay=5e-4)
    w = [O.seeded_fill(5 ^ l, n, 0.05).astype(np.float32) for l, n in enumerate(elems)]
    v = [np.zeros(n, np.float32) for n in elems]
    for x in xs:
        for l in range(len(elems)):
            x.layer_views[l].copy_(torch.from_numpy(w[l]))
    torch.cuda.synchronize()
    for k in range(3):
        for l in reversed(range(len(elems))):
            n = elems[l]
            grads = [np.random.default_rng([r, l, k]).standard_normal(n, dtype=np.float32) * np.float32(1e-2)
                     for r in range(N)]
            pieces = [split_pieces(torch.from_numpy(g).cuda(), n - 1001) for g in grads]
            stepped_layer(xs, trs, l, k, pieces)
            w[l], v[l] = O.exchange_iteration(grads, w[l], 0.01, "fast32", state=v[l], scale=1.0 / N,
                                              momentum=0.9, weight_decay=5e-4)
            for r in range(N):
                assert xs[r].layer_views[l].cpu().numpy().tobytes() == w[l].tobytes(), (N, k, l, r)
    for x in xs:
        x.close()
    world.close()


@pytest.mark.parametrize("variant", ["twoshot", "tree", "twoshot_ce", "oneshot", "oneshot_ll", "twoshot_bulk",
                                     "twoshot_l128", "twoshot_ceb", "twoshot_cet"])
def test_misaligned_gradient_views_match_oracle(cuda, variant):
    """Gradient pieces that are views at 4- and 12-byte offsets into larger buffers (not
    16-byte aligned): the kernels must fall back from the per-slab vector path to the
    element-wise piece lookup and stay bit-exact (N=4, fast32, a slab-straddling cut)."""
    N = 4
    elems = [70001, 1_200_007]
    world, trs, xs = build(N, elems, "fast32", variant, lr=0.01, momentum=0.9, weight_decay=5e-4)
    w = [O.seeded_fill(11 ^ l, n, 0.05).astype(np.float32) for l, n in enumerate(elems)]
    v = [np.zeros(n, np.float32) for n in elems]
    for x in xs:
        for l in range(len(elems)):
            x.layer_views[l].copy_(torch.from_numpy(w[l]))
    torch.cuda.synchronize()
    keep = []
    for k in range(2):
        for l in reversed(range(len(elems))):
            n = elems[l]
            grads = [np.random.default_rng([r, l, k, 3]).standard_normal(n, dtype=np.float32) * np.float32(1e-2)
                     for r in range(N)]
            cut = n // 2 + 1
            pieces = []
            for g in grads:
                a = torch.zeros(cut + 8, device="cuda")
                b = torch.zeros(n - cut + 8, device="cuda")
                a[1:1 + cut] = torch.from_numpy(g[:cut]).cuda()
                b[3:3 + n - cut] = torch.from_numpy(g[cut:]).cuda()
                pieces.append([a[1:1 + cut], b[3:3 + n - cut]])
                keep += [a, b]
            stepped_layer(xs, trs, l, k, pieces)
            w[l], v[l] = O.exchange_iteration(grads, w[l], 0.01, "fast32", state=v[l], scale=1.0 / N,
                                              momentum=0.9, weight_decay=5e-4)
            for r in range(N):
                assert xs[r].layer_views[l].cpu().numpy().tobytes() == w[l].tobytes(), (variant, k, l, r)
    for x in xs:
        x.close()
    world.close()


def test_graph_instantiated_with_node_priorities_replays_the_exchange(cuda):
    """pgx_graph_instantiate_prio / pgx_graph_launch (bench.py --graph-prio): a captured
    training step launched through the library's executable applies exactly the oracle
    update, replay after replay, like torch's own replay."""
    import ctypes

    from paper_1706_00095_b200 import _lib
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import LocalWorld

    m = _FixedGrad(40000, 6)
    layers = [(m, [m.weight, m.bias])]
    world = LocalWorld(1, inline=False)
    tr = world.transport(0)
    x = DeviceExchange(tr, [40007], mode="fast32", lr=0.05, momentum=0.9, weight_decay=1e-3)
    x.connect()
    w = torch.cat([m.weight.detach(), m.bias.detach()]).cpu().numpy()
    g = torch.cat([m.c, m.d]).cpu().numpy()
    bind = ModuleBinding(x, layers)
    v = np.zeros_like(w)

    def step():
        m().backward()
        bind.step_done()

    step()
    bind.drain()
    torch.cuda.synchronize()
    x.set_device_iteration(True, bind.k - 1)
    graph = torch.cuda.CUDAGraph(keep_graph=True)
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap), torch.cuda.graph(graph, stream=cap):
        bind.begin_step()
        step()
        bind.drain()
    torch.cuda.current_stream().wait_stream(cap)
    torch.cuda.synchronize()
    ex = ctypes.c_void_p()
    _lib.call("pgx_graph_instantiate_prio", ctypes.c_void_p(graph.raw_cuda_graph()), ctypes.byref(ex))
    s = torch.cuda.current_stream()
    for _ in range(3):
        _lib.call("pgx_graph_launch", ex, ctypes.c_void_p(s.cuda_stream))
    bind.wait_current()
    torch.cuda.synchronize()
    _lib.call("pgx_graph_exec_destroy", ex)
    for _ in range(1 + 3):  # the eager step before the capture + 3 launches (capturing runs nothing)
        w, v = O.fast32_update(w, v, g, 1.0, 0.05, 0.9, 1e-3)
    assert tr.device_status() == 0
    assert x.layer_views[0].cpu().numpy().tobytes() == w.tobytes()
    bind.remove()
    x.close()
    world.close()
