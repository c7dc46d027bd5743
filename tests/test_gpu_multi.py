"""Real multi-GPU runs: one process per GPU, CUDA-IPC peer segments, concurrent
device-side waits over NVLink.  Skipped unless >= 2 GPUs are visible."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

LENET = [520, 25050, 400500, 5010]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, world, port, variant, mode, late, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    from oracle import pipesgd_oracle as O
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import DistTransport

    try:
        tr = DistTransport(rank, world, rank, timeout_s=20.0)
        if late:  # rendezvous first; the exchange's segments are attached afterwards
            tr.barrier()
        elems = LENET + [1 << 20]
        hyper = dict(lr=0.01, momentum=0.9, weight_decay=5e-4) if mode == "fast32" else dict(lr=0.05)
        x = DeviceExchange(tr, elems, mode=mode, variant=variant, chunk_elems=16384, flags=(("allow_l128",) if "l128" in variant else ()), **hyper)
        dt = np.float32
        w = [O.seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)).astype(dt) for l, n in enumerate(elems)]
        v = [np.zeros(n, np.float32) for n in elems]
        for l in range(len(elems)):
            x.layer_views[l].copy_(torch.from_numpy(w[l]))
        torch.cuda.synchronize()
        if late:
            tr.sync_segments()
        tr.barrier()  # rendezvous: IPC handles exchanged, peers attached
        x.connect()
        comp = torch.cuda.current_stream()
        bad = []
        for k in range(4):
            for l in range(len(elems)):
                x.gate(l, k - 1) if k else None
            grads = {}
            for l in reversed(range(len(elems))):
                n = elems[l]
                gs = [O.seeded_fill(O.derived_seed(42, r, l, k), n, 1e-2).astype(dt) for r in range(world)]
                grads[l] = gs
                g = torch.from_numpy(gs[rank]).cuda()
                x.stream.wait_stream(comp)
                g.record_stream(x.stream)
                x.launch(l, k, [g])
            for l in range(len(elems)):
                if mode == "fast32":
                    w[l], v[l] = O.exchange_iteration(grads[l], w[l], 0.01, mode, state=v[l], scale=1.0 / world,
                                                      momentum=0.9, weight_decay=5e-4)
                else:
                    w[l] = O.exchange_iteration(grads[l], w[l], 0.05, mode).astype(dt)
            for l in range(len(elems)):
                x.gate(l, k)
            torch.cuda.synchronize()
            for l in range(len(elems)):
                got = x.layer_views[l].cpu().numpy()
                if variant == "nvls":  # the switch's summation order: tolerance parity (fp32 rel 1e-5)
                    if not np.allclose(got, w[l], rtol=1e-5, atol=1e-7):
                        bad.append((k, l, float(np.max(np.abs(got - w[l])))))
                elif got.tobytes() != w[l].tobytes():
                    bad.append((k, l))
        q.put((rank, bad, tr.device_status()))
        x.close()
        tr.close()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc), -1))
    dist.destroy_process_group()


def _spawn(fn, world, *args):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda t: t[0])


def _ngpu():
    """GPUs the concurrent tests span: all visible, capped at PGX_TEST_MAX_GPUS (default 4,
    the largest world these tests were run at on B200; 8-rank correctness of every variant
    is covered on one GPU by test_gpu_exchange's LocalWorld N=8 cases)."""
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    return min(n, int(os.environ.get("PGX_TEST_MAX_GPUS", "4")))


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("variant,mode", [(v, m) for v in ("twoshot", "tree", "twoshot_ce", "twoshot_cep", "oneshot", "oneshot_ll", "oneshot_l128",
                                                                    "twoshot_bulk", "twoshot_l128", "twoshot_ceb", "twoshot_cet")
                                          for m in ("ref32", "fast32")]
                         + [("nvls", "fast32")])
def test_concurrent_exchange_matches_oracle(variant, mode):
    out = _spawn(_exchange_worker, _ngpu(), variant, mode, False)
    for rank, bad, status in out:
        assert bad == [] and status == 0, (rank, bad, status)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("variant", ["twoshot", "twoshot_ce", "twoshot_cep"])
def test_exchange_created_after_rendezvous(variant):
    """DistTransport.sync_segments attaches segments created after the first barrier."""
    out = _spawn(_exchange_worker, _ngpu(), variant, "fast32", True)
    for rank, bad, status in out:
        assert bad == [] and status == 0, (rank, bad, status)


def _engine_worker(rank, world, port, pattern, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    from paper_1706_00095_b200 import harness
    from paper_1706_00095_b200.config import TrainConfig

    try:
        cfg = TrainConfig(layer_dims=(6, 9, 5), world_size=world, iterations=4, batch_size=24, dataset_size=48,
                          seed=19, epsilon=0.08, pattern=pattern, finalize_timeout_s=20.0)
        ds = harness.build_dataset(cfg, device=f"cuda:{rank}")
        res = harness.run_dist(cfg, ds, rank, rank)
        ref = harness.sequential_sgd(cfg, ds, device=f"cuda:{rank}")
        ok = all(a.tobytes() == b.tobytes() for a, b in zip(res.model, ref))
        q.put((rank, ok, res.barrier_calls))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc), -1))
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("pattern", ["pipelined", "barrier"])
def test_host_engine_over_ipc_matches_sequential(pattern):
    out = _spawn(_engine_worker, _ngpu(), pattern)
    for rank, ok, barriers in out:
        assert ok is True, (rank, ok)
        assert barriers == (0 if pattern == "pipelined" else 8)


def _lenet():
    from workloads import LeNet

    return LeNet()


def _cifar10_quick():
    from workloads import Cifar10Quick

    return Cifar10Quick()


def _model_worker(rank, world, port, which, variant, gate, q):
    """configs[0] / configs[1]: a real model trained through ModuleBinding; every step's
    exchanged weights must equal the oracle applied to the gradients the hooks saw."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    from oracle import pipesgd_oracle as O
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import DistTransport

    try:
        torch.manual_seed(0)  # identical init on every rank
        net = (_lenet() if which == "lenet" else _cifar10_quick()).cuda()
        layers = net.layers()
        if which == "lenet":
            shape, batch, hyper = (1, 28, 28), 64 // world, dict(lr=0.01, momentum=0.0, weight_decay=0.0)
        else:
            shape, batch, hyper = (3, 32, 32), 100, dict(lr=0.001, momentum=0.9, weight_decay=0.004)
        tr = DistTransport(rank, world, rank, timeout_s=20.0)
        x = DeviceExchange(tr, [sum(p.numel() for p in ps) for _, ps in layers], mode="fast32", variant=variant,
                           **hyper)
        bind = ModuleBinding(x, layers, gate=gate)
        tr.barrier()
        x.connect()
        seen = {}
        orig = x.launch

        def spy(layer, iteration, pieces, stream=None, phases=7):
            seen[layer] = torch.cat([p.detach().reshape(-1) for p in pieces]).clone()
            return orig(layer, iteration, pieces, stream, phases)

        x.launch = spy
        g = torch.Generator(device="cpu").manual_seed(42 + rank)
        w = [x.layer_views[l].cpu().numpy().copy() for l in range(len(layers))]
        v = [np.zeros_like(a) for a in w]
        bad = []
        for k in range(3):
            data = torch.randn(batch, *shape, generator=g).cuda()
            label = torch.randint(0, 10, (batch,), generator=g).cuda()
            loss = torch.nn.functional.cross_entropy(net(data), label)
            loss.backward()
            bind.step_done()
            bind.drain()
            torch.cuda.synchronize()
            for l in range(len(layers)):
                every = [None] * world
                dist.all_gather_object(every, seen[l].cpu().numpy())
                w[l], v[l] = O.exchange_iteration(every, w[l], hyper["lr"], "fast32", state=v[l],
                                                  scale=1.0 / world, momentum=hyper["momentum"],
                                                  weight_decay=hyper["weight_decay"])
                got = x.layer_views[l].cpu().numpy()
                if variant == "nvls":  # the switch's summation order: tolerance parity (fp32 rel 1e-5)
                    if not np.allclose(got, w[l], rtol=1e-5, atol=1e-6):
                        bad.append((k, l, float(np.max(np.abs(got - w[l])))))
                elif got.tobytes() != w[l].tobytes():
                    bad.append((k, l, float(np.max(np.abs(got - w[l])))))
        q.put((rank, bad, tr.device_status()))
        x.close()
        tr.close()
    except Exception as exc:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc(), -1))
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("which", ["lenet", "cifar10_quick"])
@pytest.mark.parametrize("variant,gate", [("twoshot", "layer"), ("twoshot_ce", "layer"), ("twoshot_cep", "layer"), ("tree", "layer"),
                                          ("twoshot_ce", "model"), ("nvls", "layer"), ("oneshot", "layer"), ("oneshot_ll", "layer")])
def test_real_models_match_oracle(which, variant, gate):
    world = 2 if which == "lenet" else min(4, _ngpu())
    out = _spawn(_model_worker, world, which, variant, gate)
    for rank, bad, status in out:
        assert bad == [] and status == 0, (rank, bad, status)


def _fault_worker(rank, world, port, variant, q):
    """Rank 1 stops contributing after iteration 0; rank 0's bounded device waits must expire
    and surface as TransportError instead of hanging (fault injection, test_transport_tcp.py:134-160)."""
    import time

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    from paper_1706_00095_b200.errors import TransportError
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import DistTransport

    outcome = "no error"
    try:
        tr = DistTransport(rank, world, rank, timeout_s=2.0)
        x = DeviceExchange(tr, [1 << 16], mode="fast32", variant=variant, flags=(("allow_l128",) if "l128" in variant else ()), lr=0.01)
        tr.barrier()
        x.connect()
        g = torch.ones(1 << 16, device="cuda")
        for k in range(2):
            if k == 1 and rank == 1:
                break  # the "dead" peer
            x.launch(0, k, [g])
            x.gate(0, k)
            torch.cuda.synchronize()
        t0 = time.time()
        try:
            x.check()
        except TransportError as exc:
            outcome = f"TransportError after {time.time() - t0:.1f}s: {exc}"
    except Exception as exc:  # noqa: BLE001
        outcome = repr(exc)
    q.put((rank, outcome, 0))
    dist.barrier()  # keep the peer's memory mapped until everyone is done
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("variant", ["twoshot", "twoshot_ce", "twoshot_cep", "oneshot_ll", "oneshot_l128",
                                     "twoshot_bulk", "twoshot_l128"])
def test_dead_peer_surfaces_as_transport_error(variant):
    out = _spawn(_fault_worker, 2, variant)
    assert out[0][1].startswith("TransportError"), out
    assert out[1][1] == "no error", out


def _graph_worker(rank, world, port, variant, gate, use_graph, q):
    """Several layers, one process per GPU, the whole step captured once as a CUDA graph
    (device iteration counter) and replayed: each rank's gradient is a fixed per-rank
    constant (loss = sum(w*c_r) + sum(b*d_r)), so after the replays every rank must hold
    exactly the oracle's weights for the N-rank exchange."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    from oracle import pipesgd_oracle as O
    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import DistTransport

    class Fixed(torch.nn.Module):
        def __init__(self, n, r):
            super().__init__()
            gw = torch.Generator().manual_seed(5 + n)  # same initial weights on every rank
            self.weight = torch.nn.Parameter(torch.randn(n, generator=gw).cuda())
            self.bias = torch.nn.Parameter(torch.randn(7, generator=gw).cuda())
            gg = torch.Generator().manual_seed(1000 * r + n)  # per-rank gradients
            self.c = (torch.randn(n, generator=gg) * 1e-2).cuda()
            self.d = (torch.randn(7, generator=gg) * 1e-2).cuda()

        def forward(self, x):
            return x + (self.weight * self.c).sum() + (self.bias * self.d).sum()

    try:
        sizes = [3000, 70000, 400000, 1500000]  # LL / one-shot / two-shot / copy-engine sizes at N=4
        mods = [Fixed(n, rank) for n in sizes]
        layers = [(m, [m.weight, m.bias]) for m in mods]
        tr = DistTransport(rank, world, rank, timeout_s=20.0)
        x = DeviceExchange(tr, [n + 7 for n in sizes], mode="fast32", variant=variant, flags=(("allow_l128",) if "l128" in variant else ()), lr=0.05, momentum=0.9,
                           weight_decay=1e-3)
        bind = ModuleBinding(x, layers, gate=gate)
        tr.barrier()
        x.connect()

        def step():
            y = torch.zeros((), device="cuda")
            for m in mods:
                y = m(y)
            y.backward()
            bind.step_done()

        w0 = [torch.cat([m.weight.detach(), m.bias.detach()]).cpu().numpy() for m in mods]
        for _ in range(2):
            step()
        bind.drain()
        torch.cuda.synchronize()
        if use_graph:
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
        else:
            for _ in range(3):
                step()
            bind.drain()
        torch.cuda.synchronize()
        # oracle: 5 exchanges (2 eager steps + 3 replays; capturing runs nothing) of every
        # rank's fixed gradient
        grads = []
        for n in sizes:
            per = []
            for r in range(world):
                gg = torch.Generator().manual_seed(1000 * r + n)
                c = (torch.randn(n, generator=gg) * 1e-2).numpy()
                d = (torch.randn(7, generator=gg) * 1e-2).numpy()
                per.append(np.concatenate([c, d]).astype(np.float32))
            grads.append(per)
        bad = []
        for l, n in enumerate(sizes):
            w, v = w0[l].copy(), np.zeros_like(w0[l])
            for _ in range(5):
                w, v = O.exchange_iteration(grads[l], w, 0.05, "fast32", state=v, scale=1.0 / world,
                                            momentum=0.9, weight_decay=1e-3)
            got = x.layer_views[l].cpu().numpy()
            if got.tobytes() != w.tobytes():
                bad.append((l, float(np.max(np.abs(got - w)))))
        q.put((rank, bad, tr.device_status()))
        bind.remove()
        x.close()
        tr.close()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc), -1))
    dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("variant,gate", [("auto", "layer"), ("auto", "model"), ("twoshot", "layer"),
                                          ("twoshot_ce", "layer"), ("twoshot_cep", "model"), ("tree", "layer"),
                                          ("oneshot", "layer"), ("oneshot_ll", "model"), ("oneshot_l128", "layer"),
                                          ("twoshot_bulk", "layer"), ("twoshot_bulk", "model"),
                                          ("twoshot_l128", "model"), ("twoshot_ceb", "layer"), ("twoshot_cet", "layer")])
def test_graph_replay_multi_gpu_matches_oracle(variant, gate):
    out = _spawn(_graph_worker, _ngpu(), variant, gate, True)
    for rank, bad, status in out:
        assert bad == [] and status == 0, (rank, bad, status)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("variant", ["auto", "twoshot"])
def test_eager_chain_multi_gpu_matches_oracle(variant):
    out = _spawn(_graph_worker, _ngpu(), variant, "layer", False)
    for rank, bad, status in out:
        assert bad == [] and status == 0, (rank, bad, status)
