"""One layer's exchange for N ranks emulated on ONE GPU, phases launched in dependency order
(push of every rank, then every owner), so each exchange kernel can be profiled by ncu
without spinning on a peer (single-GPU hazard rule, tests/test_gpu_exchange.py).  The
kernels under ncu are the product kernels with the production plan for that layer
(variant, chunk, grid); "peer" stores land in this GPU's HBM, so DRAM bytes and
instruction-level evidence are real while NVLink counters are not (tools/ncu_rank0.sh
covers those on real peers).

    python tools/ncu_stepped.py --world 4 --elems 37752832 --variant twoshot --iters 3
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1706_00095_b200 import _lib
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import LocalWorld

    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=4)
    ap.add_argument("--elems", type=int, default=37752832)  # AlexNet fc6
    ap.add_argument("--variant", default="twoshot")
    ap.add_argument("--mode", default="fast32")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--ctas", type=int, default=0)
    args = ap.parse_args()
    N = args.world
    world = LocalWorld(N, inline=False)
    trs = [world.transport(r) for r in range(N)]
    xs = [DeviceExchange(tr, [args.elems], mode=args.mode, variant=args.variant, chunk_elems=16384, lr=0.01,
                         momentum=0.9, weight_decay=5e-4, max_ctas=args.ctas,
                         flags=("allow_l128",) if args.variant == "oneshot_l128" else ()) for tr in trs]
    for x in xs:
        x.connect()
    g = [[torch.randn(args.elems - 4096, device="cuda") * 1e-3, torch.randn(4096, device="cuda") * 1e-3]
         for _ in range(N)]
    for k in range(args.iters):
        for r in range(N):
            xs[r].launch(0, k, g[r], stream=trs[r].stream, phases=_lib.PHASE_PUSH)
        torch.cuda.synchronize()
        for r in range(N):
            xs[r].launch(0, k, g[r], stream=trs[r].stream, phases=_lib.PHASE_OWNER)
            torch.cuda.synchronize()
        for r in range(N):
            xs[r].gate(0, k, stream=trs[r].stream)
        torch.cuda.synchronize()
    assert all(tr.device_status() == 0 for tr in trs)
    print({"variant": args.variant, "world": N, "elems": args.elems, "plan": xs[0].layer_plan(0),
           "bytes": xs[0].layer_bytes(0)})
    for x in xs:
        x.close()
    world.close()


if __name__ == "__main__":
    main()
