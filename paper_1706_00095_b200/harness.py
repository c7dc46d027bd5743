"""Launchers and the single-process device reference run (reference harness.py, sgd.py:72-108).

* :func:`run_local` — every rank is a thread of this process, all on one GPU, over
  :class:`LocalWorld` (the ``run_inproc`` analog, harness.py:53-91).
* :func:`run_dist` — this process is one rank of a ``torch.distributed`` job, one
  GPU per rank, peers attached with CUDA IPC (the ``run_tcp`` analog; the launcher is
  ``torchrun``).
* :func:`sequential_sgd` — one process plays every rank with the device fold
  (``pgx_tree_reduce``) and device update (``pgx_master_update``): the analog of the
  reference's oracle optimizer, used by tests to pin the distributed engine.
"""

from __future__ import annotations

import threading

import torch

from . import _lib, net
from .config import TrainConfig
from .engine import BarrierRank, PipelinedRank, RankResult, batch_indices, shard_bounds
from .errors import VerificationError
from .ops import tree_reduce
from .topology import build_reduction_tree
from .transport import DistTransport, LocalWorld


def _rank_class(pattern: str):
    return PipelinedRank if pattern == "pipelined" else BarrierRank


def build_dataset(cfg: TrainConfig, device="cuda"):
    dtype = torch.float64 if cfg.dtype == "f64" else torch.float32
    return net.make_synthetic_dataset(cfg.seed, cfg.dataset_size, cfg.specs(), cfg.input_scale, dtype, device)


def run_local(config: TrainConfig, dataset, device: int = 0, record: bool = False) -> list[RankResult]:
    """All ranks as threads of this process on one GPU; returns results by rank."""
    world = LocalWorld(config.world_size, device=device, inline=True)
    results: list = [None] * config.world_size
    failures: list = []

    def body(rank: int) -> None:
        try:
            tr = world.transport(rank)
            rec = None
            if record:
                from .timeline import Recorder
                rec = Recorder(rank)
            results[rank] = _rank_class(config.pattern)(config, dataset, tr, rec).run()
        except BaseException as exc:  # noqa: BLE001 - reported below
            failures.append((rank, exc))
            world.abort_barrier()

    threads = [threading.Thread(target=body, args=(r,), name=f"rank-{r}", daemon=True)
               for r in range(config.world_size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=config.finalize_timeout_s * (config.iterations + 2))
    world.close()
    if failures:
        rank, exc = sorted(failures, key=lambda f: f[0])[0]
        raise exc
    if any(r is None for r in results):
        raise VerificationError("a rank did not finish")
    return results


def run_dist(config: TrainConfig, dataset, rank: int, device: int, group=None, recorder=None) -> RankResult:
    """This process's rank of a multi-GPU run (peers on other GPUs, CUDA IPC)."""
    tr = DistTransport(rank, config.world_size, device, group, timeout_s=config.finalize_timeout_s)
    try:
        return _rank_class(config.pattern)(config, dataset, tr, recorder).run()
    finally:
        tr.close()


def sequential_sgd(config: TrainConfig, dataset, on_iteration=None, device="cuda") -> list:
    """One process plays all ranks (sgd.py:72-108) with the device fold and update."""
    dtype = torch.float64 if config.dtype == "f64" else torch.float32
    specs = config.specs()
    model = net.init_model(config.seed, specs, dtype, device)
    tree = build_reduction_tree(config.world_size)
    for k in range(config.iterations):
        idx = batch_indices(config.seed, k, config.batch_size, len(dataset))
        partials, loss0 = [], 0.0
        for r in range(config.world_size):
            lo, hi = shard_bounds(config.batch_size, config.world_size, r)
            x, t = dataset.take(idx[lo:hi])
            grads, loss = net.backward(specs, model, x, t)
            partials.append(grads)
            if r == 0:
                loss0 = float(loss)
        red = tree_reduce(partials, tree, dtype=dtype)
        fn = "pgx_master_update_f64" if dtype == torch.float64 else "pgx_master_update_f32"
        for l in range(len(specs)):
            _lib.call(fn, model[l].data_ptr(), red[l].data_ptr(), float(config.epsilon), model[l].data_ptr(),
                      model[l].numel(), torch.cuda.current_stream().cuda_stream)
        if on_iteration is not None:
            on_iteration(k, model, loss0)
    torch.cuda.synchronize()
    return [m.cpu().numpy() for m in model]


def verify_against_reference(config: TrainConfig, dataset, results) -> None:
    ref = sequential_sgd(config, dataset)
    for res in results:
        for l, (got, want) in enumerate(zip(res.model, ref)):
            if got.tobytes() != want.tobytes():
                raise VerificationError(f"rank {res.rank} layer {l} differs from the sequential reference")
