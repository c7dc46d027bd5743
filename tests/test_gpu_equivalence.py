"""Distributed device runs reproduce the single-process run bit for bit, and the
device exchange reproduces the REFERENCE's own models when fed its gradients
(reference tests/test_equivalence.py analogs)."""

import numpy as np
import pytest
import torch

from oracle import pipesgd_oracle as O

pytestmark = pytest.mark.gpu


def problem(world_size, **kw):
    from paper_1706_00095_b200 import harness
    from paper_1706_00095_b200.config import TrainConfig

    cfg = TrainConfig(layer_dims=(6, 9, 5), world_size=world_size, iterations=6, batch_size=24, dataset_size=48,
                      seed=19, epsilon=0.08, finalize_timeout_s=20.0).replace(**kw)
    return cfg, harness.build_dataset(cfg)


def same(results, ref):
    for res in results:
        for l, (a, b) in enumerate(zip(res.model, ref)):
            assert a.tobytes() == b.tobytes(), f"rank {res.rank} layer {l}"


@pytest.mark.parametrize("world_size", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("pattern", ["pipelined", "barrier"])
def test_matches_sequential(cuda, world_size, pattern):
    from paper_1706_00095_b200 import harness

    cfg, ds = problem(world_size, pattern=pattern)
    same(harness.run_local(cfg, ds), harness.sequential_sgd(cfg, ds))


@pytest.mark.parametrize("kw", [{"chunk_bytes": 64, "iterations": 3}, {"dtype": "f32"},
                                {"layer_dims": (4, 16, 16, 2), "iterations": 4}, {"layer_dims": (5, 1, 4)}])
def test_variants_match_sequential(cuda, kw):
    from paper_1706_00095_b200 import harness

    cfg, ds = problem(4, **kw)
    same(harness.run_local(cfg, ds), harness.sequential_sgd(cfg, ds))


def test_barrier_counts_and_fold_accounting(cuda):
    from paper_1706_00095_b200 import harness

    cfg, ds = problem(4)
    assert all(r.barrier_calls == 0 for r in harness.run_local(cfg, ds))
    assert all(r.barrier_calls == 2 * cfg.iterations for r in harness.run_local(cfg.replace(pattern="barrier"), ds))
    cfg8, ds8 = problem(8, iterations=2)
    res = harness.run_local(cfg8, ds8)
    for l in range(len(cfg8.specs())):
        assert sum(r.fold_counts[l] for r in res) == 7 * 2


def test_sequential_matches_cpu_oracle_on_device_gradients(cuda):
    """Same device gradients, exchange arithmetic on the CPU oracle: identical bits."""
    from paper_1706_00095_b200 import harness, net
    from paper_1706_00095_b200.engine import batch_indices, shard_bounds

    cfg, ds = problem(4, iterations=3)
    specs = cfg.specs()
    model = [m.cpu().numpy() for m in net.init_model(cfg.seed, specs)]
    for k in range(cfg.iterations):
        idx = batch_indices(cfg.seed, k, cfg.batch_size, len(ds))
        dm = [torch.from_numpy(m).cuda() for m in model]
        parts = []
        for r in range(cfg.world_size):
            lo, hi = shard_bounds(cfg.batch_size, cfg.world_size, r)
            x, t = ds.take(idx[lo:hi])
            g, _ = net.backward(specs, dm, x, t)
            parts.append([gi.cpu().numpy() for gi in g])
        for l in range(len(specs)):
            model[l] = O.exchange_iteration([p[l] for p in parts], model[l], cfg.epsilon, "ref64")
    ref = harness.sequential_sgd(cfg, ds)
    for a, b in zip(model, ref):
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("ws", [1, 2, 3, 4, 8])
def test_reference_gradients_through_device_engine(cuda, golden, ws):
    """Drive PipelinedRank turn by turn with the REFERENCE's per-rank gradients
    (tests/golden, produced by pipesgd itself) and compare with its final model."""
    from paper_1706_00095_b200.config import TrainConfig
    from paper_1706_00095_b200.engine import PipelinedRank
    from paper_1706_00095_b200.transport import LocalWorld

    arr, meta = golden
    e = [x for x in meta["e2e"] if x["world_size"] == ws][0]
    cfg = TrainConfig(layer_dims=(6, 9, 5), world_size=ws, iterations=e["iterations"], batch_size=24,
                      dataset_size=48, seed=19, epsilon=e["epsilon"], finalize_timeout_s=10.0)
    world = LocalWorld(ws, inline=True)
    ranks = [PipelinedRank(cfg, None, world.transport(r)) for r in range(ws)]
    L = len(e["layers"])
    for r in ranks:  # reference initial model (identical to init_model by construction)
        for l in range(L):
            assert r.model_views[l].cpu().numpy().tobytes() == arr[f"e2e{ws}_k0_w{l}"].tobytes()
    for k in range(e["iterations"]):
        for r in ranks:
            r.begin_iteration(k)
        for l in range(L - 1, -1, -1):
            for r in reversed(ranks):
                r.run_turn(l, torch.from_numpy(arr[f"e2e{ws}_k{k}_r{r.rank}_l{l}"]))
        for r in ranks:
            r.finalize_iteration()
    torch.cuda.synchronize()
    for r in ranks:
        for l in range(L):
            assert r.model_views[l].cpu().numpy().tobytes() == arr[f"e2e{ws}_final_l{l}"].tobytes()
    assert [r.fold_counts for r in ranks] == e["fold_counts"]
    world.close()


def test_loss_decreases(cuda):
    from paper_1706_00095_b200 import harness

    cfg, ds = problem(4, iterations=30, epsilon=0.05)
    losses = harness.run_local(cfg, ds)[0].losses
    assert np.mean(losses[-5:]) < np.mean(losses[:5])
