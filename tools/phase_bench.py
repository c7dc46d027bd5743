"""Per-phase throughput of the exchange kernels on N GPUs driven from ONE process (host-stepped:
every phase is launched on all ranks only when the flags it waits on are already set, so no
kernel spins).  Separates raw transfer throughput from cross-rank skew.

    python tools/phase_bench.py [--mb 256] [--variants twoshot,twoshot_ce,tree]
"""
import argparse, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_00095_b200 import _lib
from paper_1706_00095_b200.exchange import DeviceExchange
from paper_1706_00095_b200.transport import LocalWorld

ap = argparse.ArgumentParser()
ap.add_argument("--mb", type=float, default=256)
ap.add_argument("--variants", default="twoshot,twoshot_ce,tree")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--ctas", type=int, default=0)
args = ap.parse_args()
N = torch.cuda.device_count()
S = int(args.mb * 2 ** 20 / 4)
for v in args.variants.split(","):
    world = LocalWorld(N, inline=False, devices=list(range(N)))
    trs = [world.transport(r) for r in range(N)]
    xs = [DeviceExchange(tr, [S], mode="fast32", variant=v, lr=0.01, momentum=0.9, max_ctas=args.ctas) for tr in trs]
    for x in xs:
        x.connect()
    gs = [torch.randn(S, device=f"cuda:{r}") * 1e-3 for r in range(N)]
    phases = ([_lib.PHASE_PUSH, _lib.PHASE_OWNER] if v != "tree" else [_lib.PHASE_PUSH, _lib.PHASE_DOWN])
    res = {p: [] for p in phases}
    for it in range(args.iters + 1):
        for ph in phases:
            order = range(N) if not (v == "tree" and ph == _lib.PHASE_PUSH) else reversed(range(N))
            evs = []
            for r in order:
                with torch.cuda.device(r):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(trs[r].stream)
                    xs[r].launch(0, it, [gs[r]], stream=trs[r].stream, phases=ph)
                    xs[r].join(0, trs[r].stream)
                    e1.record(trs[r].stream)
                    evs.append((r, e0, e1))
                if v == "tree":  # tree phases depend rank to rank: finish each before the next
                    torch.cuda.synchronize(r)
            for r in range(N):
                torch.cuda.synchronize(r)
            if it:
                res[ph].append(max(e0.elapsed_time(e1) for _, e0, e1 in evs))
    for r in range(N):
        xs[r].gate(0, args.iters, stream=trs[r].stream)
        torch.cuda.synchronize(r)
        assert trs[r].device_status() == 0
    own = S // N * 4
    for ph, ts in res.items():
        ms = statistics.median(ts)
        out_bytes = (N - 1) * own  # bytes each rank sends in this phase (two-shot)
        print(json.dumps({"variant": v, "n_gpus": N, "phase": {1: "push/up", 2: "owner", 4: "down"}[ph],
                          "layer_bytes": S * 4, "ms": ms, "out_GBps_per_rank": out_bytes / (ms / 1e3) / 1e9}), flush=True)
    for x in xs:
        x.close()
    world.close()
