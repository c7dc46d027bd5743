"""Gradient-exchange sweep (BASELINE.json configs[4]): per-layer sizes 4 KB..256 MB at N GPUs,
two-shot vs tree vs NCCL all-reduce (comparison only), fused update on.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/sweep.py [--max-mb 256] [--ctas 0]

Each point: device flag barrier, a busy kernel (--hold-us) queued on the stream so the host's
enqueue latency is hidden, then ONE layer exchange (launch + gate) timed with CUDA events on
the exchange stream, median of --iters after --warmup, max over ranks.
busBW convention: 2(N-1)/N * bytes / t.  Prints one JSON line per point on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mb", type=float, default=256)
    ap.add_argument("--min-kb", type=float, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--align", type=int, default=1,
                    help="1: a device flag barrier on the timed stream right before the start event, so "
                         "ranks start within one flag round trip (host wake-up skew excluded; NCCL too)")
    ap.add_argument("--hold-us", type=float, default=300.0,
                    help="busy kernel queued ahead of each timed launch (excludes host enqueue latency; 0 = off)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=16384)
    ap.add_argument("--variants", default="twoshot,twoshot_ce,tree,nccl")
    ap.add_argument("--mode", default="fast32")
    ap.add_argument("--xflags", default="", help="comma-separated exchange flags (exchange.FLAGS)")
    args = ap.parse_args()

    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import DistTransport

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nccl = dist.new_group(backend="nccl") if world > 1 else None

    sizes = []
    b = int(args.min_kb * 1024)
    while b <= args.max_mb * 2 ** 20:
        sizes.append(b)
        b *= 4
    esz = 8 if args.mode == "ref64" else 4  # ref64: the reference's native f64 elements
    elems = [s // esz for s in sizes]
    variants = args.variants.split(",")
    out = []
    tr = DistTransport(rank, world, local, timeout_s=30.0)
    xs = {}
    seg = 16
    for v in variants:
        if v in ("twoshot", "tree", "twoshot_ce", "twoshot_cep", "nvls", "oneshot", "oneshot_ll", "oneshot_l128",
                 "twoshot_bulk", "twoshot_l128", "twoshot_ceb", "twoshot_cet"):
            xs[v] = DeviceExchange(tr, elems, mode=args.mode, variant=v, chunk_elems=args.chunk, lr=0.01,
                                   momentum=0.9, weight_decay=5e-4, seg_base=seg, max_ctas=args.ctas,
                                   flags=tuple(f for f in args.xflags.split(",") if f)
                                   + (("allow_l128",) if "l128" in v else ()))
            seg += 2
    tr.barrier()
    for x in xs.values():
        x.connect()

    HOLD_CYCLES = int(args.hold_us * 1965)  # SM clock 1965 MHz

    def tmax(ms):
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for li, n in enumerate(elems):
        g = torch.randn(n, device=dev, dtype=torch.float64 if esz == 8 else torch.float32) * 1e-3
        for v in variants:
            times = []
            for it in range(args.warmup + args.iters):
                tr.barrier()  # device flag barrier: every rank starts together
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                # keep the stream busy while the host enqueues, so the events bracket device
                # time only (not the Python/ctypes launch latency), for every variant and NCCL
                hold = torch.cuda.current_stream() if v == "nccl" else xs[v].stream
                if HOLD_CYCLES:
                    with torch.cuda.stream(hold):
                        torch.cuda._sleep(HOLD_CYCLES)
                if args.align and world > 1:  # device barrier right before e0: no start skew
                    tr.barrier_async(hold)
                if v == "nccl":
                    s = torch.cuda.current_stream()
                    e0.record(s)
                    dist.all_reduce(g, group=nccl)
                    e1.record(s)
                else:
                    x = xs[v]
                    k = it + 1000 * 0
                    e0.record(x.stream)
                    x.launch(li, k + li * 0, [g])
                    x.join(li, x.stream)
                    x.gate(li, k, stream=x.stream)
                    e1.record(x.stream)
                torch.cuda.synchronize()
                if it >= args.warmup:
                    times.append(e0.elapsed_time(e1))
            ms = tmax(statistics.median(times))
            nbytes = n * esz
            bus = 2 * (world - 1) / world * nbytes / (ms / 1e3) / 1e9 if world > 1 else None
            rec = {"n_gpus": world, "variant": v, "bytes": nbytes, "ms": ms, "busbw_gbs": bus,
                   "frac_of_770": bus / 770.0 if bus else None, "ctas": args.ctas, "chunk_elems": args.chunk,
                   "update": ("fused " + args.mode) if v != "nccl" else "none (all-reduce only)", "elem_bytes": esz,
                   "hold_us": args.hold_us, "aligned_start": bool(args.align), "xflags": args.xflags or None}
            if rank == 0:
                print(json.dumps(rec), flush=True)
            out.append(rec)
    # keep each exchange's epochs consistent: every layer got warmup+iters launches with k = it
    for x in xs.values():
        x.close()
    tr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
