"""NVLink bytes per exchange from the GPUs' own link counters (NVML field values
NVLINK_THROUGHPUT_DATA_TX/RX and RAW_TX/RX, summed over the links), beside the exchange's
algorithmic bytes and CUDA-event time.  This is the multi-rank evidence for "achieved
NVLink GB/s": ncu must not wrap a multi-rank command (B200_PROFILING.md), while NVML reads
the same hardware counters without touching the kernels.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_counters.py \
        [--mb 144] [--variants twoshot,twoshot_bulk,twoshot_ce,nccl] [--reps 50]

Per rank and variant: reps back-to-back exchanges of one layer (device barrier before each),
counters read before / after on the rank's own device; one JSON line per (variant, rank).
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


def nvml_handle(dev: int):
    import pynvml

    pynvml.nvmlInit()
    p = torch.cuda.get_device_properties(dev)
    bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    try:
        return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
    except Exception:  # noqa: BLE001
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(dev)


# (name, NVML field, unit bytes): per-link byte counters (COUNT_*, Blackwell) and the older
# throughput counters (KiB); whichever the driver answers is used
FIELDS = (("XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", 1), ("RCV_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", 1),
          ("DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", 1024),
          ("DATA_RX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX", 1024),
          ("RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", 1024), ("RAW_RX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX", 1024))


def read_counters(nv, h) -> tuple[dict, dict]:
    """Bytes per field summed over every link that answers, and the NVML return codes seen."""
    out = {f: 0 for f, _, _ in FIELDS}
    codes: dict = {}
    for link in range(18):
        try:
            vals = nv.nvmlDeviceGetFieldValues(h, [(getattr(nv, fid), link) for _, fid, _ in FIELDS])
        except Exception as exc:  # noqa: BLE001
            codes.setdefault("exception", repr(exc))
            continue
        for (f, _, unit), v in zip(FIELDS, vals):
            rc = int(getattr(v, "nvmlReturn", -1))
            codes.setdefault(f, set()).add(rc)
            if rc == 0:
                out[f] += int(v.value.ullVal) * unit
    return out, {k: sorted(v) if isinstance(v, set) else v for k, v in codes.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=144.0)  # AlexNet fc6 is 151 MB
    ap.add_argument("--variants", default="twoshot,twoshot_bulk,twoshot_ce,nccl")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--ctas", type=int, default=0)
    args = ap.parse_args()

    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import DistTransport

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nccl = dist.new_group(backend="nccl")
    nv, h = nvml_handle(local)
    n = int(args.mb * 2 ** 20) // 4
    tr = DistTransport(rank, world, local, timeout_s=30.0)
    xs, seg = {}, 16
    for v in args.variants.split(","):
        if v != "nccl":
            xs[v] = DeviceExchange(tr, [n], mode="fast32", variant=v, lr=0.01, momentum=0.9, weight_decay=5e-4,
                                   seg_base=seg, max_ctas=args.ctas)
            seg += 2
    tr.barrier()
    for x in xs.values():
        x.connect()
    g = torch.randn(n, device=dev) * 1e-3
    for v in args.variants.split(","):
        def one(k):
            if v == "nccl":
                dist.all_reduce(g, group=nccl)
                return
            x = xs[v]
            x.launch(0, k, [g], stream=x.stream)
            x.join(0, x.stream)
            x.gate(0, k, stream=x.stream)

        stream = torch.cuda.current_stream() if v == "nccl" else xs[v].stream
        for k in range(3):  # warm
            one(k)
        torch.cuda.synchronize()
        tr.barrier()
        c0, codes = read_counters(nv, h)
        times = []
        for k in range(3, 3 + args.reps):
            tr.barrier_async(stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one(k)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        tr.barrier()
        c1, _ = read_counters(nv, h)
        per = {f: (c1[f] - c0[f]) / args.reps for f, _, _ in FIELDS}
        ms = statistics.median(times)
        alg = 2 * (world - 1) / world * n * 4
        rec = {"variant": v, "rank": rank, "n_gpus": world, "bytes": n * 4, "ms_median": ms,
               "algorithmic_out_bytes": alg, "nvlink_bytes_per_exchange": per,
               "tx_over_algorithmic": (per["XMIT_BYTES"] or per["DATA_TX"]) / alg if alg else None,
               "achieved_tx_gbs": (per["XMIT_BYTES"] or per["DATA_TX"]) / (ms / 1e3) / 1e9, "nvml_return_codes": codes,
               "achieved_busbw_gbs": alg / (ms / 1e3) / 1e9,
               "counter_source": "NVML NVLINK_COUNT_{XMIT,RCV}_BYTES and NVLINK_THROUGHPUT_*, summed over links",
               "note": "median event time includes the device barrier skew; counters cover every rep"}
        allr = [None] * world
        dist.all_gather_object(allr, rec)
        if rank == 0:
            for r in allr:
                print(json.dumps(r), flush=True)
    for x in xs.values():
        x.close()
    tr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
