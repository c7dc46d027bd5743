"""Exchanges for N ranks emulated on ONE GPU, phases launched in dependency order (push of
every rank, then every owner), so each exchange kernel can be profiled by ncu or checked by
compute-sanitizer without spinning on a peer (single-GPU hazard rule,
tests/test_gpu_exchange.py).  The kernels are the product kernels with the production plan
for the layer (variant, chunk, grid); "peer" stores land in this GPU's HBM, so DRAM bytes and
instruction-level evidence are real while NVLink counters are not (tools/nvlink_counters.py
reads those on real peers).  With --check every rank's weights are compared bit for bit with
the oracle after every iteration.

    python tools/ncu_stepped.py --world 4 --elems 37752832 --variants twoshot,twoshot_bulk --iters 3
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_1706_00095_b200 import _lib
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import LocalWorld

    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=4)
    ap.add_argument("--elems", default="37752832")  # AlexNet fc6; comma-separated layer list
    ap.add_argument("--variants", default="twoshot")
    ap.add_argument("--mode", default="fast32")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--devices", default="", help="rank->GPU map, e.g. 0,1: peers' stores then cross NVLink")
    args = ap.parse_args()
    N = args.world
    elems = [int(e) for e in args.elems.split(",")]
    devs = [int(d) for d in args.devices.split(",")] if args.devices else [0] * N
    if len(devs) != N:
        raise SystemExit("--devices needs one GPU per rank")

    def sync():  # every GPU the ranks live on (torch.cuda.synchronize covers the current one only)
        for d in sorted(set(devs)):
            torch.cuda.synchronize(d)

    for variant in args.variants.split(","):
        world = LocalWorld(N, inline=False, devices=devs if args.devices else None)
        trs = [world.transport(r) for r in range(N)]
        xs = [DeviceExchange(tr, elems, mode=args.mode, variant=variant, chunk_elems=16384, lr=0.01,
                             momentum=0.9, weight_decay=5e-4, max_ctas=args.ctas,
                             flags=("allow_l128",) if "l128" in variant else ()) for tr in trs]
        for x in xs:
            x.connect()
            x.model.zero_()
        sync()
        if args.check:
            from oracle import pipesgd_oracle as O
            w = [np.zeros(n, np.float32) for n in elems]
            v = [np.zeros(n, np.float32) for n in elems]
        for k in range(args.iters):
            for l in reversed(range(len(elems))):
                n = elems[l]
                gh = [np.random.default_rng([r, l, k]).standard_normal(n, dtype=np.float32) * np.float32(1e-3)
                      for r in range(N)]
                cut = n - min(4096, max(1, n // 8))
                g = [[torch.from_numpy(a[:cut]).to(f"cuda:{devs[r]}"), torch.from_numpy(a[cut:]).to(f"cuda:{devs[r]}")]
                     for r, a in enumerate(gh)]
                if variant == "tree":  # children (higher ranks) before parents, then back down
                    for r in reversed(range(N)):
                        xs[r].launch(l, k, g[r], stream=trs[r].stream, phases=_lib.PHASE_PUSH)
                        sync()
                    for r in range(N):
                        xs[r].launch(l, k, g[r], stream=trs[r].stream, phases=_lib.PHASE_DOWN)
                        sync()
                elif variant == "twoshot_l128":  # push, owner, install
                    for ph in (_lib.PHASE_PUSH, _lib.PHASE_OWNER, _lib.PHASE_DOWN):
                        for r in range(N):
                            xs[r].launch(l, k, g[r], stream=trs[r].stream, phases=ph)
                        sync()
                else:
                    for r in range(N):
                        xs[r].launch(l, k, g[r], stream=trs[r].stream, phases=_lib.PHASE_PUSH)
                    sync()
                    for r in range(N):
                        xs[r].launch(l, k, g[r], stream=trs[r].stream, phases=_lib.PHASE_OWNER)
                        sync()
                for r in range(N):
                    xs[r].gate(l, k, stream=trs[r].stream)
                sync()
                if args.check:
                    w[l], v[l] = O.exchange_iteration(gh, w[l], 0.01, "fast32", state=v[l], scale=1.0 / N,
                                                      momentum=0.9, weight_decay=5e-4)
                    for r in range(N):
                        assert xs[r].layer_views[l].cpu().numpy().tobytes() == w[l].tobytes(), (variant, k, l, r)
        assert all(tr.device_status() == 0 for tr in trs)
        print({"variant": variant, "world": N, "elems": elems, "plan": [xs[0].layer_plan(l) for l in range(len(elems))],
               "bytes": [xs[0].layer_bytes(l) for l in range(len(elems))], "checked": args.check}, flush=True)
        for x in xs:
            x.close()
        world.close()


if __name__ == "__main__":
    main()
