"""Per-work-item device timeline of one exchange (pgx_xchg_set_trace; ONESHOT and
TWOSHOT_BULK are instrumented): where the time of a layer goes (push / fence+flag / wait /
fold), every rank.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/trace_oneshot.py [--kb 1024]
        [--variant oneshot|twoshot_bulk] [--ctas 0]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_00095_b200 import _lib  # noqa: E402
from paper_1706_00095_b200.exchange import DeviceExchange  # noqa: E402
from paper_1706_00095_b200.transport import DistTransport  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kb", type=int, default=1024)
    ap.add_argument("--chunk", type=int, default=16384)
    ap.add_argument("--variant", default="oneshot")
    ap.add_argument("--ctas", type=int, default=0)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = args.kb * 256
    tr = DistTransport(rank, world, local, timeout_s=20.0)
    x = DeviceExchange(tr, [n], mode="fast32", variant=args.variant, chunk_elems=args.chunk, lr=0.01, momentum=0.9,
                       max_ctas=args.ctas)
    tr.barrier()
    x.connect()
    g = torch.randn(n, device="cuda") * 1e-3
    ch = x.layer_plan(0)[0]
    sl = ((n + world - 1) // world + 3) // 4 * 4  # two-shot shard (pgx_xchg_create)
    C_ = -(-n // ch) if args.variant == "oneshot" else -(-sl // ch)
    items = (world - 1) * C_ + C_
    buf = torch.zeros(items * 8, dtype=torch.int64, device="cuda")
    out = []
    for it in range(8):
        traced = it >= 5
        _lib.call("pgx_xchg_set_trace", x.handle, C.c_void_p(buf.data_ptr() if traced else 0))
        buf.zero_()
        tr.barrier()
        with torch.cuda.stream(x.stream):
            torch.cuda._sleep(300 * 1965)
        tr.barrier_async(x.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(x.stream)
        x.launch(0, it, [g], stream=x.stream)
        x.join(0, x.stream)
        x.gate(0, it, stream=x.stream)
        e1.record(x.stream)
        torch.cuda.synchronize()
        if traced:
            t = buf.view(items, 8).cpu().tolist()
            t0 = min(r[0] for r in t if r[0])
            push = [(r[0] - t0, r[1] - t0, r[2] - t0) for r in t[: (world - 1) * C_]]
            own = [(r[0] - t0, r[1] - t0, r[2] - t0) for r in t[(world - 1) * C_:]]
            out.append({"rank": rank, "event_us": e0.elapsed_time(e1) * 1e3,
                        "push_claim_us": [min(p[0] for p in push) / 1e3, max(p[0] for p in push) / 1e3],
                        "push_stores_done_us": statistics.median(p[1] for p in push) / 1e3,
                        "push_flag_done_us_med_max": [statistics.median(p[2] for p in push) / 1e3,
                                                      max(p[2] for p in push) / 1e3],
                        "owner_claim_us": [min(o[0] for o in own) / 1e3, max(o[0] for o in own) / 1e3],
                        "owner_wait_done_us_med_max": [statistics.median(o[1] for o in own) / 1e3,
                                                       max(o[1] for o in own) / 1e3],
                        "owner_end_us_med_max": [statistics.median(o[2] for o in own) / 1e3,
                                                 max(o[2] for o in own) / 1e3],
                        "items": items, "chunk": x.layer_plan(0)[0], "ctas": x.layer_plan(0)[1],
                        "variant": args.variant, "kb": args.kb,
                        "push_item_us_med": statistics.median(p[2] - p[0] for p in push) / 1e3,
                        "owner_fold_us_med": statistics.median(o[2] - o[1] for o in own) / 1e3,
                        "owner_acc_us_med": [statistics.median(r[k] for r in t[(world - 1) * C_:]) / 1e3
                                             for k in (4, 5, 6)],
                        "owner_rounds": statistics.median(r[7] for r in t[(world - 1) * C_:]),
                        "owner_acc": "TWOSHOT_BULK: fold round (loads+update+local stores), store issue, "
                                     "output-ring wait (us per item)"})
    allr = [None] * world
    dist.all_gather_object(allr, out)
    if rank == 0:
        for r in allr:
            for d in r:
                print(json.dumps(d))
    x.close()
    tr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
