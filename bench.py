"""Benchmark: AlexNet (B=256 global, synthetic 227x227) data-parallel SGD with the
per-layer device exchange — images/sec at N GPUs (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W]                 # our arm
    python bench.py --impl reference [--gpus N ...]                  # CPU reference arm
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A step = one training iteration: forward + backward of AlexNet on this rank's
256/N images (PyTorch/cuDNN, bf16 autocast, fp32 master weights), during which
every layer's gradient is exchanged and the fused momentum-SGD update applied by
libpgx kernels as soon as that layer's gradient is final; the next forward of a
layer waits only for that layer's new weights.  One JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GLOBAL_BATCH = 256  # AlexNet, BASELINE.json configs[2]
ALEXNET_LAYERS = [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]
METRIC = "AlexNet images/sec (B=256 global, synthetic 227x227), per-layer gradient exchange"


def wl_of(args):
    from workloads import WORKLOADS

    return WORKLOADS[args.workload]


def global_batch(wl, world):
    return wl["global_batch"] if "global_batch" in wl else wl["per_gpu_batch"] * world
NVLINK_PEAK_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (900 nominal)
L128_BAND = ((1 << 16) + 1, 1 << 20)  # = exchange.L128_BAND (kept import-free for the reference arm)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--workload", default="alexnet", choices=["alexnet", "googlenet", "lenet", "cifar10_quick"])
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="pgx", choices=["pgx", "reference"])
    p.add_argument("--variant", default="auto", choices=["twoshot", "tree", "twoshot_ce", "twoshot_cep", "twoshot_bulk", "nvls", "oneshot", "auto", "nccl_bulk",
                            "ddp"],
                   help="nccl_bulk / ddp are comparison rows (NCCL on the path), not the product")
    p.add_argument("--chunk-elems", type=int, default=16384)
    p.add_argument("--gate", default="auto", choices=["auto", "layer", "model"],
                   help="per-layer forward gates, or one whole-model gate per step (auto: model if > 16 layers)")
    p.add_argument("--max-ctas", type=int, default=0)
    p.add_argument("--large", choices=("ce", "cep", "sm", "bulk", "ceb", "cet"), default="ce",
                   help="auto policy for layers >= 1M elements: copy-engine or SM two-shot")
    p.add_argument("--large-ctas", type=int, default=0, help="CTA cap of the large layers' launches (0 = auto)")
    p.add_argument("--large-chunk-elems", type=int, default=0, help="chunk of the large layers (0 = --chunk-elems)")
    p.add_argument("--low-priority-from", type=int, default=0,
                   help="layers with at least this many elements launch on a normal-priority stream (0 = off)")
    p.add_argument("--xflags", default="", help="comma-separated exchange flags (exchange.FLAGS), e.g. bulk_lean")
    p.add_argument("--overlap-ctas", type=int, default=16,
                   help="CTA cap of the small layers whose exchange overlaps the backward (all but layer 0); "
                        "0 = off (profiles/r6k: GoogLeNet N=4 +1.8 %%, AlexNet N=4 +0.9 %%)")
    p.add_argument("--ce-parts", type=int, default=0, help="copy-engine owner pipelining depth (0 = library default 4)")
    p.add_argument("--overlap-exposed", type=int, default=1,
                   help="how many of the first layers (emitted last by backward) keep the full grid")
    p.add_argument("--l128", default="%d:%d" % L128_BAND,
                   help="LO:HI elements sent by the 128-byte-line two-shot (adds allow_l128); '' = off")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="eager steps instead of a captured CUDA graph")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--timeline", default="")
    p.add_argument("--graph-prio", action="store_true",
                   help="diagnostic: instantiate the step graph with the capture streams' priorities on its "
                        "nodes (pgx_graph_instantiate_prio); dropout masks then repeat across replays")
    p.add_argument("--trace-graph", action="store_true",
                   help="diagnostic: bracket every layer's exchange with events inside the step graph and "
                        "report them (graph_trace) relative to the step start / backward end")
    p.add_argument("--per-gpu-batch", type=int, default=0,
                   help="diagnostic only: override 256/N (the line is then not the headline config)")
    return p.parse_args()


def cpu_info():
    try:
        model = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")][0]
    except Exception:  # noqa: BLE001
        model = "unknown"
    return model, len(os.sched_getaffinity(0))


# ------------------------------------------------------------------ CPU side
# The reference is CPU code: its exchange engine is pipesgd's PipelinedRank over InprocWorld
# (pipelined.py:44-80), which bench.py runs from baseline/_ref (the reference package,
# installed unmodified; it travels to the GPU box) and restates in C (oracle/pgx_oracle.c,
# threaded, the "port").  The networks' forward/backward is not part of the reference; the
# CPU training step below runs it in PyTorch-CPU on the FULL batch (no extrapolation).
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def _mk_batch(wl, n, seed=0):
    import torch

    g = torch.Generator().manual_seed(seed)
    x = torch.randn(n, wl.get("channels", 3), wl["image"], wl["image"], generator=g)
    y = torch.randint(0, wl.get("classes", 1000), (n,), generator=g)
    return x, y


def cpu_fwd_bwd_ms(net, x, y) -> float:
    t0 = time.perf_counter()
    loss = net.loss(net(x), y)
    loss.backward()
    net.zero_grad(set_to_none=True)
    return (time.perf_counter() - t0) * 1e3


def port_exchange(world: int, sizes, iters: int = 3, threads: int | None = None):
    """(median ms, ExchangeWorld) of the C port of the reference's exchange iteration (tree
    fold in the binomial order, fused update, broadcast) at `world` ranks on host threads."""
    from oracle import c_oracle as CO

    threads = threads or cpu_info()[1]
    ex = CO.ExchangeWorld(world, sizes, fast_fill=True)
    ex.iteration("fast32", threads=threads)  # warm (page faults)
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        ex.iteration("fast32", lr=0.01, mu=0.9, wd=5e-4, threads=threads)
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts), ex


def reference_engine_ms(world: int, sizes, iters: int = 2) -> dict:
    """The reference's own exchange engine (pipesgd PipelinedRank.begin_iteration / run_turn /
    finalize_iteration over InprocWorld, zero latency, f64 — pipelined.py:44-80) at the given
    per-layer sizes (DenseLayerSpec(S-1, 1) so param_count = S).  Rank threads are
    GIL-serialised and numpy is single-threaded: about one core.  Last iteration's time, max
    over the rank threads."""
    import threading

    import numpy as np

    if not os.path.isdir(os.path.join(REF_PATH, "pipesgd")):
        return {"unavailable": f"reference package not installed at {REF_PATH}"}
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        from pipesgd.engine import PipelinedRank, TrainConfig
        from pipesgd.net import DenseLayerSpec
        from pipesgd.transport import InprocWorld
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"cannot import the reference: {exc!r}"}
    cfg = TrainConfig(layer_dims=(2, 1), world_size=world, iterations=iters, batch_size=world,
                      chunk_bytes=65536, finalize_timeout_s=600.0)
    specs = [DenseLayerSpec(int(n) - 1, 1, "identity") for n in sizes]
    cfg.specs = lambda: specs
    w = InprocWorld(world)
    try:
        ranks = [PipelinedRank(cfg, None, w.transport(r)) for r in range(world)]
        rng = np.random.default_rng(0)
        grads = [rng.standard_normal(int(n)) * 1e-3 for n in sizes]  # values do not change the work
        times = [[0.0] * iters for _ in range(world)]

        def body(r):
            rk = ranks[r]
            for k in range(iters):
                t0 = time.perf_counter()
                rk.begin_iteration(k)
                for l in reversed(range(len(sizes))):
                    rk.run_turn(l, grads[l])
                rk.finalize_iteration()
                times[r][k] = time.perf_counter() - t0

        ths = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    finally:
        w.close()
    per_it = [max(times[r][k] for r in range(world)) * 1e3 for k in range(iters)]
    return {"ms": per_it[-1], "iterations": iters, "all_ms": [round(t, 3) for t in per_it],
            "engine": "pipesgd PipelinedRank over InprocWorld (baseline/_ref, f64, ~1 core)"}


def cpu_step(world: int, wl_name: str, *, steps: int | None = None, seconds: float | None = None,
             warmup: int = 1) -> dict:
    """The training step on the host: the full global batch through PyTorch-CPU fp32 fwd+bwd
    (all threads) plus one exchange iteration of the C port at `world` ranks, every counted
    step measured (no sample scaling)."""
    import torch

    from workloads import WORKLOADS

    model_name, ncpu = cpu_info()
    torch.set_num_threads(ncpu)
    wl = WORKLOADS[wl_name]
    net = wl["cls"]()
    gb = global_batch(wl, world)
    sizes = [sum(p.numel() for p in ps) for _, ps in net.layers()]
    x, y = _mk_batch(wl, gb)
    ex_ms, ex = port_exchange(world, sizes, iters=1)
    for _ in range(warmup):
        cpu_fwd_bwd_ms(net, x, y)
    fb, xc = [], []
    t_end = time.perf_counter() + (seconds or 1e9)
    while (steps is None or len(fb) < steps) and (time.perf_counter() < t_end or not fb):
        fb.append(cpu_fwd_bwd_ms(net, x, y))
        t0 = time.perf_counter()
        ex.iteration("fast32", lr=0.01, mu=0.9, wd=5e-4, threads=ncpu)
        xc.append((time.perf_counter() - t0) * 1e3)
    tot = [a + b for a, b in zip(fb, xc)]
    ms = sum(tot) / len(tot)
    return {"value": gb / (ms / 1e3), "unit": "images/s", "cores": ncpu, "kind": "port",
            "sample": f"{len(fb)} full steps; each: {wl_name} fwd+bwd of the whole {gb}-image batch in PyTorch-CPU "
                      f"fp32 (not part of the reference, which has no conv nets) + one exchange iteration of the "
                      f"{sum(sizes):,} fp32 params at world {world} by the C port of the reference's tree fold + "
                      f"update + broadcast (oracle/pgx_oracle.c, {ncpu} threads); cpu {model_name}",
            "ms_per_step": ms, "ms_fwd_bwd": statistics.median(fb), "ms_exchange": statistics.median(xc),
            "exchange_only_images_per_s": gb / (statistics.median(xc) / 1e3), "steps_measured": len(fb)}


def exchange_by_world(sizes, worlds=(2, 4, 8)) -> dict:
    """CPU exchange per iteration at each world size: the C port and the reference's own
    engine (BASELINE.md §2 measured 1.1 / 3.6 / 16.8 s for AlexNet)."""
    out = {}
    for w in worlds:
        ms, ex = port_exchange(w, sizes, iters=3)
        del ex
        out[str(w)] = {"port_ms": ms, "port_threads": cpu_info()[1], "reference_engine": reference_engine_ms(w, sizes)}
    return out


def xflags_of(args) -> tuple:
    fl = tuple(f for f in args.xflags.split(",") if f)
    return fl + (("allow_l128",) if args.l128 and "allow_l128" not in fl else ())


def l128_of(args) -> tuple:
    if not args.l128:
        return (0, 0)
    lo, hi = args.l128.split(":")
    return (int(lo), int(hi))


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    wl = wl_of(args)
    sizes = [sum(p.numel() for p in ps) for _, ps in wl["cls"]().layers()]
    r = cpu_step(world, args.workload, steps=args.steps, warmup=max(1, min(args.warmup, 2)))
    ref = reference_engine_ms(world, sizes) if world > 1 or args.workload != "alexnet" else \
        reference_engine_ms(1, sizes)
    cfg = workload_config(world, args)
    cfg.update({"fwd_bwd": "PyTorch-CPU fp32, full batch every step", "exchange": "C port of the reference's "
                "exchange (tree fold + update + broadcast), all host threads", "step": "eager (CPU)"})
    for k in ("chunk_elems", "large_layers", "gate"):
        cfg.pop(k, None)
    cb = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "ms_fwd_bwd", "ms_exchange",
                            "exchange_only_images_per_s", "steps_measured")}
    cb["reference_engine_exchange"] = ref
    line = {"metric": wl["metric"], "value": r["value"], "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": cfg, "cpu_baseline": cb,
            "e2e": {"value": r["value"], "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(world, args):
    wl = wl_of(args)
    gb = global_batch(wl, world)
    name = {"alexnet": "alexnet_b256_synthetic_227", "googlenet": "googlenet_b32pergpu_synthetic_224",
            "lenet": "lenet5_b64_synthetic_28", "cifar10_quick": "cifar10_quick_b100pergpu_synthetic_32"}[args.workload]
    model = {"alexnet": "AlexNet (BVLC, grouped conv, LRN)",
             "googlenet": "GoogLeNet (BVLC, both aux heads, 64 param layers)",
             "lenet": "LeNet-5 (Caffe lenet_train_test)", "cifar10_quick": "cifar10_quick (Caffe)"}[args.workload]
    h = wl["hyper"]
    return {"workload": name, "model": model,
            "global_batch": gb, "per_gpu_batch": gb // world,
            "image": [wl.get("channels", 3), wl["image"], wl["image"]],
            "parallelism": f"dp{world}", "exchange": args.variant, "update": f"fast32 momentum SGD lr {h['lr']} mu {h['momentum']} "
            f"wd {h['weight_decay']} scale 1/N", "fwd_bwd": "PyTorch cuDNN bf16 autocast, fp32 master weights/grads",
            "l2": "working set > L2 (244 MB fp32 weights + 244 MB grads + activations per step)"
                  if args.workload == "alexnet" else "per-step working set (weights, grads, activations)",
            "chunk_elems": args.chunk_elems, "large_layers": {"variant": args.large, "ctas": args.large_ctas,
                                                               "chunk_elems": args.large_chunk_elems},
            "gate": args.gate, "step": "CUDA graph replay" if not args.no_graph else "eager",
            "exchange_flags": args.xflags or None, "l128_range": args.l128 or None,
            "overlap_ctas": args.overlap_ctas, "overlap_exposed": args.overlap_exposed,
            "graph_prio": args.graph_prio or None,
            "ce_parts": args.ce_parts or None}


# ------------------------------------------------------------------ model
def alexnet():
    from workloads import AlexNet

    return AlexNet()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML every 10 ms on a
    thread (a timed region can be ~0.2 s, too short for nvidia-smi's 200 ms loop), falling
    back to `nvidia-smi -lms 200` when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple] = []
        self._nv = None
        self._stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.device)
            bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:  # noqa: BLE001
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def start(self):
        try:
            self._nv = self._nvml_handle()
            self._t = threading.Thread(target=self._poll_nvml, daemon=True)
            self._t.start()
            return
        except Exception:  # noqa: BLE001
            self._nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _poll_nvml(self):
        nv, h = self._nv
        bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((float(sm), float(mx), {k for k, b in bits.items() if r & b}))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.01)

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self._nv is not None:
            self._stop.set()
            self._t.join(timeout=2)
            sm = [a for a, _, _ in self.samples]
            reasons = set().union(*[r for _, _, r in self.samples]) if self.samples else set()
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": max(b for _, b, _ in self.samples) if self.samples else None,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "NVML, 10 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi, 200 ms"}


# ------------------------------------------------------------------ our arm
def pgx_arm(args):
    import torch
    import torch.distributed as dist

    from paper_1706_00095_b200.exchange import DeviceExchange, ModuleBinding
    from paper_1706_00095_b200.transport import DistTransport

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)  # plumbing: handles + timing max
    torch.backends.cudnn.benchmark = True
    torch.manual_seed(1234 + rank)

    wl = wl_of(args)
    model = wl["cls"]().to(dev)
    sizes = [sum(p.numel() for p in ps) for _, ps in model.layers()]
    tr = DistTransport(rank, world, local, timeout_s=60.0)
    xchg = DeviceExchange(tr, sizes, mode="fast32", variant=args.variant, chunk_elems=args.chunk_elems,
                          scale=1.0 / world, max_ctas=args.max_ctas,
                          low_priority_from=args.low_priority_from or None, large=args.large,
                          large_ctas=args.large_ctas, large_chunk_elems=args.large_chunk_elems,
                          flags=xflags_of(args), l128_range=l128_of(args), overlap_ctas=args.overlap_ctas,
                          overlap_exposed=args.overlap_exposed, ce_parts=args.ce_parts,
                          **wl["hyper"])
    gate = args.gate if args.gate != "auto" else ("model" if len(sizes) > 16 else "layer")
    bind = ModuleBinding(xchg, model.layers(), gate=gate)
    if world > 1:  # identical initial weights everywhere: broadcast rank 0's (plumbing, untimed)
        flat = xchg.model.cpu()
        dist.broadcast(flat, 0)
        xchg.model.copy_(flat.to(dev))
        torch.cuda.synchronize()
    tr.barrier()      # rendezvous: every rank's segments attached over CUDA IPC
    xchg.connect()

    B = args.per_gpu_batch or global_batch(wl, world) // world
    IMG = wl["image"]
    gb = B * world  # images per step, whole job
    g = torch.Generator().manual_seed(42 + rank)
    CH_IN, NCLS = wl.get("channels", 3), wl.get("classes", 1000)
    host_x = torch.randint(0, 256, (B, CH_IN, IMG, IMG), dtype=torch.uint8, generator=g).pin_memory()
    host_y = torch.randint(0, NCLS, (B,), dtype=torch.int64, generator=g).pin_memory()
    dev_x, dev_y = host_x.to(dev), host_y.to(dev)
    loss_host = torch.zeros(max(args.steps, 1), dtype=torch.float32).pin_memory()

    def step(xb, yb):
        xin = xb.to(torch.bfloat16, memory_format=torch.channels_last).sub_(128.0).mul_(1.0 / 64.0)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = model(xin)
        loss = model.loss(out, yb)
        loss.backward()
        bind.step_done()
        return loss

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step(dev_x, dev_y)
    bind.drain()
    torch.cuda.synchronize()
    L_DOM = max(range(len(sizes)), key=lambda l: sizes[l])  # the dominant (largest) layer; AlexNet: fc6

    # ---- capture one training step as a CUDA graph (epochs from the device counter) ----
    graph = None
    bind.timed_layers = {L_DOM}  # bracket the dominant layer's exchange with (external) events
    if args.trace_graph:
        bind.timed_layers = set(range(len(sizes)))
    bind.events.clear()
    gmarks = None
    if not args.no_graph:
        k_before_capture = bind.k
        xchg.set_device_iteration(True, bind.k - 1)
        graph = torch.cuda.CUDAGraph(keep_graph=args.graph_prio)
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream())
        c0 = xchg.launch_count()
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                bind.begin_step()
                if args.trace_graph:
                    gmarks = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
                    gmarks[0].record()
                static_loss = step(dev_x, dev_y)
                if gmarks:
                    gmarks[1].record()  # the compute stream is past the backward
                bind.drain()  # joins every exchange stream back into the capture
                if gmarks:
                    gmarks[2].record()
        per_step_launches = xchg.launch_count() - c0
        torch.cuda.current_stream().wait_stream(cap)
        torch.cuda.synchronize()
        replays = [0]
        prio_exec = None
        if args.graph_prio:
            import ctypes

            from paper_1706_00095_b200 import _lib
            ex = ctypes.c_void_p()
            _lib.call("pgx_graph_instantiate_prio", ctypes.c_void_p(graph.raw_cuda_graph()), ctypes.byref(ex))
            prio_exec = ex

        def run_step(xb=None, yb=None):
            if xb is not None:
                dev_x.copy_(xb, non_blocking=True)
                dev_y.copy_(yb, non_blocking=True)
            if prio_exec is not None:
                _lib.call("pgx_graph_launch", prio_exec, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
            else:
                graph.replay()
            replays[0] += 1
            return static_loss

        def finish():
            bind.wait_current()
    else:
        def run_step(xb=None, yb=None):
            return step(dev_x if xb is None else xb, dev_y if yb is None else yb)

        def finish():
            bind.drain()

    def timed(fn, k):
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(k):
            fn(i)
        finish()  # the last iteration's weights are installed everywhere
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---- device-resident timed region (value) ----
    clocks = ClockSampler(local)
    clocks.start()
    n0 = xchg.launch_count()
    ms = timed(lambda i: run_step(), args.steps)
    launches = xchg.launch_count() - n0
    clk = clocks.stop()
    if graph is not None:  # launches inside replays are not counted by the host: count one captured step
        launches = per_step_launches * args.steps
    value = gb * args.steps / (ms / 1e3)

    # ---- end-to-end through the public API: host batch in, loss out ----
    e2e = None
    if not args.no_e2e:
        # every step's batch crosses from pinned host memory inside the timed region, as a
        # data loader would deliver it: step i+1's H2D copy (copy engine, own stream) is
        # issued before step i's compute so it overlaps it; a 13 us D2D copy installs it
        # into the graph's static input once step i has finished reading the previous one
        h2d = torch.cuda.Stream(device=dev)
        stage = [(torch.empty_like(dev_x), torch.empty_like(dev_y)) for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        consumed = [None, None]

        def prefetch(j):
            b = j % 2
            with torch.cuda.stream(h2d):
                if consumed[b] is not None:
                    h2d.wait_event(consumed[b])
                stage[b][0].copy_(host_x, non_blocking=True)
                stage[b][1].copy_(host_y, non_blocking=True)
                ready[b].record(h2d)

        def e2e_step(i):
            b = i % 2
            cur = torch.cuda.current_stream(dev)
            if i == 0:
                prefetch(0)
            cur.wait_event(ready[b])
            dev_x.copy_(stage[b][0], non_blocking=True)
            dev_y.copy_(stage[b][1], non_blocking=True)
            consumed[b] = torch.cuda.Event()
            consumed[b].record(cur)
            if i + 1 < args.steps:
                prefetch(i + 1)
            loss = run_step()
            loss_host[i % loss_host.numel()].copy_(loss.detach(), non_blocking=True)
        ms_e2e = timed(e2e_step, args.steps)
        h2d = (host_x.numel() * host_x.element_size() + host_y.numel() * host_y.element_size()) * world
        e2e = {"value": gb * args.steps / (ms_e2e / 1e3), "unit": "images/s",
               "input_pipeline": "pinned host batch -> device by copy engine on a side stream, one step "
                                 "ahead (double-buffered), inside the timed region; loss read back every step",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4 * world, "ms_per_step": ms_e2e / args.steps,
               "final_loss": float(loss_host[(args.steps - 1) % loss_host.numel()])}

    graph_trace = None
    # ---- dominant-layer exchange time inside steps: the events captured in the graph (or
    # recorded by every eager step) bracket that layer's exchange on its streams ----
    durs = []
    if graph is not None:
        for _ in range(9):  # a few more replays, each read back (the captured events hold the last one)
            run_step()
            torch.cuda.synchronize()
            a, b_ = bind.events[L_DOM][0]
            durs.append(a.elapsed_time(b_))
        if gmarks:  # the last replay's per-layer exchange spans on the device clock
            z = gmarks[0]
            graph_trace = {"backward_end_ms": z.elapsed_time(gmarks[1]), "step_end_ms": z.elapsed_time(gmarks[2]),
                           "layers": [[l, round(z.elapsed_time(bind.events[l][0][0]), 4),
                                       round(z.elapsed_time(bind.events[l][0][1]), 4)]
                                      for l in sorted(bind.events)],
                           "note": "[layer, exchange launch (gradient ready), this rank's part done] ms from the "
                                   "start of the captured step; diagnostic run (--trace-graph)"}
        bind.wait_current()
        torch.cuda.synchronize()
        bind.k = k_before_capture + replays[0]  # continue the epoch sequence eagerly after the replays
        xchg.set_device_iteration(False, 0)
    else:
        durs = [a.elapsed_time(b_) for a, b_ in bind.events.get(L_DOM, [])]
    bind.timed_layers = set()

    # ---- timeline: a few traced eager steps, reference CSV schema + overlap ----
    timeline = trace_timeline(args, bind, model, step, dev_x, dev_y, rank, world)
    timeline.update(pipelined_vs_barrier(bind, step, dev_x, dev_y, world))

    # ---- the same forward + backward with the exchange switched off (hooks drop the
    # gradients, gates pass): what the step would cost with a free exchange ----
    alone = fwd_bwd_alone(args, bind, model, dev_x, dev_y, dev, world, barrier)
    alone["exchange_overhead_ms"] = ms / args.steps - alone["ms_per_step"]
    alone["step_over_fwd_bwd"] = (ms / args.steps) / alone["ms_per_step"]

    # ---- per-layer exchange in isolation (same launch, no concurrent backward, host enqueue
    # latency hidden behind a busy kernel so the events bracket device time): every rank,
    # device flag barrier before each, launch -> own part done -> gate on all arrivals.  The
    # dominant layer feeds the roofline; every layer >= 4 MB is reported against NVLink
    # (north star: >= 70 % for such layers).  Runs last: it advances only these layers' epochs. ----
    HOLD_CYCLES = 300 * 1965  # ~300 us busy kernel ahead of each isolated launch

    def isolated(l, reps=10):
        pieces = [torch.randn_like(p) * 1e-3 for p in model.layers()[l][1]]
        ts = []
        for i in range(reps):
            tr.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(xchg.stream):  # hide the host's enqueue latency (device time only)
                torch.cuda._sleep(HOLD_CYCLES)
            if world > 1:
                tr.barrier_async(xchg.stream)  # ranks start within one flag round trip
            e0.record(xchg.stream)
            xchg.launch(l, bind.k + i, pieces, stream=xchg.stream)
            xchg.join(l, xchg.stream)
            xchg.gate(l, bind.k + i, stream=xchg.stream)
            e1.record(xchg.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms_ = statistics.median(ts)
        if world > 1:
            t = torch.tensor([ms_])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_ = float(t.item())
        return ms_

    # whole-model exchange alone (every layer in emission order, back to back, no backward):
    # the exchange-only time per iteration, beside the CPU reference's (exchange_only below)
    def whole_model(reps=10):
        pieces = [[torch.randn_like(p) * 1e-3 for p in ps] for _, ps in model.layers()]
        ts = []
        for i in range(reps):
            tr.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(xchg.stream):
                torch.cuda._sleep(HOLD_CYCLES)
            if world > 1:
                tr.barrier_async(xchg.stream)
            e0.record(xchg.stream)
            for l in reversed(range(len(sizes))):
                s_l = xchg.stream_for(l)
                if s_l is not xchg.stream:
                    s_l.wait_stream(xchg.stream)
                xchg.launch(l, bind.k + i, pieces[l], stream=s_l)
            for l in range(len(sizes)):
                xchg.join(l, xchg.stream)
            xchg.gate_all(bind.k + i, stream=xchg.stream)
            e1.record(xchg.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        bind.k += reps
        ms_ = statistics.median(ts)
        if world > 1:
            t = torch.tensor([ms_])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_ = float(t.item())
        return ms_

    xchg_ms = whole_model()
    iso = [isolated(L_DOM)]
    by_layer = []
    if world > 1:
        for l, n in enumerate(sizes):
            if n * 4 < (4 << 20):
                continue
            ms_l = iso[0] if l == L_DOM else isolated(l)
            busbw = 2 * (world - 1) / world * n * 4 / (ms_l / 1e3) / 1e9
            by_layer.append({"layer": l, "bytes": n * 4, "variant": xchg.variants[l], "chunk_elems": xchg.layer_plan(l)[0],
                             "isolated_ms": ms_l,
                             "busbw_gbs": busbw, "frac_of_770": busbw / NVLINK_PEAK_GBS})

    # the same large layers through the SM two-shot kernel (not the in-step choice at N>1 when
    # the copy-engine variant is picked: SM stores are faster alone but steal SMs from cuDNN)
    by_layer_sm = []
    if world > 1 and by_layer and any(r["variant"] != "twoshot" for r in by_layer):
        alt = DeviceExchange(tr, sizes, mode="fast32", variant="twoshot", chunk_elems=args.chunk_elems,
                             scale=1.0 / world, seg_base=24, **wl["hyper"])
        tr.sync_segments()
        alt.connect()
        for r in by_layer:
            l, n = r["layer"], sizes[r["layer"]]
            pieces = [torch.randn_like(p) * 1e-3 for p in model.layers()[l][1]]
            ts = []
            for i in range(12):
                tr.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(alt.stream):
                    torch.cuda._sleep(HOLD_CYCLES)
                tr.barrier_async(alt.stream)
                e0.record(alt.stream)
                alt.launch(l, i, pieces)
                alt.join(l, alt.stream)
                alt.gate(l, i, stream=alt.stream)
                e1.record(alt.stream)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            t = torch.tensor([statistics.median(ts)])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_l = float(t.item())
            busbw = 2 * (world - 1) / world * n * 4 / (ms_l / 1e3) / 1e9
            by_layer_sm.append({"layer": l, "bytes": n * 4, "variant": "twoshot", "chunk_elems": alt.layer_plan(l)[0],
                                "isolated_ms": ms_l,
                                "busbw_gbs": busbw, "frac_of_770": busbw / NVLINK_PEAK_GBS})
        tr.barrier()
        alt.close()

    nvl, hbm = xchg.layer_bytes(L_DOM)
    avg = statistics.median(durs) if durs else None  # median: one replay can catch a host hiccup
    kname = {"twoshot": "k_twoshot", "twoshot_ce": "k_owner_local + copy-engine transfers",
             "twoshot_cep": "k_twoshot owner items + copy-engine reduce-scatter",
             "twoshot_bulk": "k_twoshot_bulk (TMA bulk copies, capped grid)",
             "twoshot_ceb": "k_twoshot_bulk owner slabs (TMA all-gather) + copy-engine reduce-scatter",
             "twoshot_cet": "k_owner_tma (TMA-fed fold + update, capped grid) + copy-engine reduce-scatter / all-gather",
             "tree": "k_tree_up/k_tree_down", "nvls": "k_nvls (multimem)",
             "oneshot": "k_oneshot", "twoshot_l128": "k_twoshot_l128 (128-byte lines, fence-free)",
             "oneshot_ll": "k_oneshot_ll", "oneshot_l128": "k_oneshot_l128"}[xchg.variants[L_DOM]]
    what = "%s, layer %d (%d params): fold + fused momentum update%s" % (
        kname, L_DOM, sizes[L_DOM], " + reduce-scatter/all-gather over NVLink" if world > 1 else "")
    measured_in = (("median of CUDA events captured in the step graph, %d replays after the timed region" % len(durs))
                   if graph is not None else "CUDA events in every timed eager step")
    traffic, traffic_nvl, traffic_src = ncu_traffic(kname.split()[0], world, sizes[L_DOM])
    roof = None
    if avg and world == 1:  # one GPU: the fused update is an HBM stream
        peak, peak_src = hbm_peak()
        ach = hbm / (avg / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": what, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "algorithmic_bytes_per_launch": hbm, "avg_launch_ms_in_step": avg, "in_step_ms_samples": [round(d, 4) for d in durs],
                "peak_source": peak_src, "launch_share_of_step": avg / (ms / args.steps), "measured_in": measured_in,
                "traffic_source": traffic_src}
        if iso:
            roof["isolated_launch_ms"] = statistics.median(iso)
            roof["isolated_achieved"] = hbm / (statistics.median(iso) / 1e3) / 1e9
            roof["isolated_frac"] = roof["isolated_achieved"] / peak
    elif avg:  # several GPUs: the layer's exchange is bound by this GPU's NVLink out-bandwidth
        iso_ms = statistics.median(iso)
        ach = nvl / (avg / 1e3) / 1e9
        roof = {"bound": "nvlink", "kernel": what, "achieved": ach, "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                "frac": ach / NVLINK_PEAK_GBS, "traffic": traffic, "algorithmic_bytes_per_launch": nvl,
                "bytes": "2(N-1)/N x layer bytes leave this GPU (reduce-scatter + all-gather)",
                "avg_launch_ms_in_step": avg, "in_step_ms_samples": [round(d, 4) for d in durs], "launch_share_of_step": avg / (ms / args.steps),
                "peak_source": "B200_PROFILING.md measured NVLink peer copy per direction (900 nominal)",
                "measured_in": measured_in + "; in-step time includes waiting for the slowest rank's gradient",
                "isolated_ms": iso_ms, "isolated_achieved": nvl / (iso_ms / 1e3) / 1e9,
                "isolated_frac": nvl / (iso_ms / 1e3) / 1e9 / NVLINK_PEAK_GBS,
                "hbm_bytes_per_launch": hbm, "traffic_nvlink_tx": traffic_nvl, "traffic_source": traffic_src}
    line = {"metric": wl["metric"], "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (uint8 images, random labels; random-init "
            "weights)", "config": workload_config(world, args), "roofline": roof, "clocks": clk,
            "gpu_launches": launches, "e2e": e2e, "cuda_graph": graph is not None, "timeline": timeline, "fwd_bwd_alone": alone,
            "graph_trace": graph_trace,
            "exchange_by_layer": by_layer or None, "exchange_by_layer_sm_twoshot": by_layer_sm or None}
    # ---- exchange only: the whole model's exchange per iteration, GPU (device time, every layer
    # back to back, no backward) vs the CPU reference at the same world size (rank 0 only) ----
    xo = {"gpu_ms": xchg_ms, "world": world, "model_bytes_fp32": 4 * sum(sizes),
          "gpu_measured": "all layers launched back to back in emission order + whole-model gate, device time, "
                          "median of 10, max over ranks"}
    if rank == 0 and not args.no_cpu_baseline:
        port_ms, ex = port_exchange(world, sizes, iters=3)
        del ex
        xo.update({"cpu_port_ms": port_ms, "cpu_port_threads": cpu_info()[1],
                   "port_over_gpu": port_ms / xchg_ms})
        if world > 1 or args.workload != "alexnet":
            ref = reference_engine_ms(world, sizes)
            xo["cpu_reference_engine"] = ref
            if "ms" in ref:
                xo["reference_engine_over_gpu"] = ref["ms"] / xchg_ms
    line["exchange_only"] = xo
    if args.per_gpu_batch:
        line["config"]["per_gpu_batch"] = B
        line["config"]["global_batch"] = gb
        line["config"]["diagnostic"] = "per-GPU batch overridden; not the headline configuration"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_step(world, args.workload, seconds=args.cpu_seconds)
        line["cpu_baseline"]["exchange_by_world"] = exchange_by_world(sizes, wl.get("cpu_worlds", (2, 4, 8)))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()  # rank 0's CPU timings ran while the peers waited; close together
    if tr.device_status() != 0:
        raise SystemExit(f"device status {tr.device_status()} (timeout in a device wait)")
    xchg.close()
    tr.close()
    if world > 1:
        dist.destroy_process_group()


def fwd_bwd_alone(args, bind, model, dev_x, dev_y, dev, world, barrier, reps=10):
    """Forward + backward of the benched model alone (ModuleBinding.disabled: no exchange
    launch, no gate, gradients dropped), replayed from its own CUDA graph like the step,
    device time per step, max over ranks."""
    import torch
    import torch.distributed as dist

    def body():
        xin = dev_x.to(torch.bfloat16, memory_format=torch.channels_last).sub_(128.0).mul_(1.0 / 64.0)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = model(xin)
        model.loss(out, dev_y).backward()

    bind.disabled = True
    try:
        for _ in range(3):
            body()
        torch.cuda.synchronize()
        run = body
        if not args.no_graph:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
                body()
            torch.cuda.current_stream().wait_stream(s)
            run = g.replay
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        if world > 1:
            tt = torch.tensor([t])
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
    finally:
        bind.disabled = False
    return {"ms_per_step": t, "reps": reps,
            "measured": "same model and inputs, exchange hooks and gates disabled, "
                        + ("CUDA-graph replays" if not args.no_graph else "eager steps") + ", max over ranks"}


def trace_timeline(args, bind, model, step, dev_x, dev_y, rank, world, steps=3):
    """Per-layer exchange spans vs per-layer backward spans on the device clock (CUDA events),
    in the reference's timeline schema (timeline.py:34) and its overlap ratio (timeline.py:137).
    backward_layer(l) runs from the gradient w.r.t. the layer's output being ready (a tensor
    hook on the module's output = the start of the layer's own backward kernels) to the layer's
    parameter gradients being final (the exchange trigger, pipelined.py:91-95); send_trigger(l)
    from that point to this rank's part of the layer exchange being done."""
    import torch

    from paper_1706_00095_b200.timeline import Recorder, compute_overlap, write_timeline_csv

    rec = Recorder(rank)
    bind.trace = []
    marks, starts, handles = [], [], []

    def fwd_hook(l):
        def hook(_m, _inp, out):
            t = out[0] if isinstance(out, tuple) else out
            if torch.is_tensor(t) and t.requires_grad:
                k = bind.k

                def on_grad(_g):
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record()
                    starts.append((k, l, ev))
                t.register_hook(on_grad)
        return hook

    for l, (mod, _) in enumerate(model.layers()):
        handles.append(mod.register_forward_hook(fwd_hook(l)))
    try:
        for _ in range(steps):
            k = bind.k
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            xin = dev_x.to(torch.bfloat16, memory_format=torch.channels_last).sub_(128.0).mul_(1.0 / 64.0)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                out = model(xin)
            loss = model.loss(out, dev_y)
            ev[1].record()
            loss.backward()
            ev[2].record()
            bind.step_done()
            marks.append((k, ev))
        bind.drain()
        torch.cuda.synchronize()
    finally:
        for h in handles:
            h.remove()
    t0 = marks[0][1][0]
    ns = lambda e: int(t0.elapsed_time(e) * 1e6)  # noqa: E731
    ready = {(k, l): r0 for k, l, r0, _ in bind.trace}
    for k, ev in marks:
        rec.record("forward", k, -1, ns(ev[0]), ns(ev[1]))
    nlayer = 0
    for k, l, ev in starts:
        if (k, l) in ready:
            a, b = ns(ev), ns(ready[(k, l)])
            rec.record("backward_layer", k, l, min(a, b), b)
            nlayer += 1
    tails = []
    for k, l, r0, e1 in bind.trace:
        rec.record("send_trigger", k, l, ns(r0), ns(e1))
    for k, ev in marks:
        ends = [ns(e1) for kk, l, r0, e1 in bind.trace if kk == k]
        tails.append(max(0, max(ends) - ns(ev[2])) / 1e6 if ends else 0.0)
    bind.trace = None
    path = args.timeline or ""
    if path:
        write_timeline_csv(rec.events, path.replace("{rank}", str(rank)))
    return {"overlap_ratio": compute_overlap(rec.events).overlap_ratio, "steps_traced": steps,
            "backward_layer_spans": nlayer,
            "definition": "comm time inside per-layer backward spans (layer output-grad ready -> param grads "
                          "final) or forward, / comm time (timeline.py:137-175)",
            "exchange_tail_after_backward_ms": statistics.mean(tails), "schema": "timeline.py:34 CSV",
            "csv": path or None}


def pipelined_vs_barrier(bind, step, dev_x, dev_y, world, steps=6):
    """Wall time per eager step, pipelined (exchange launched from each layer's hook) vs the
    phase-separated schedule (every exchange launched after the whole backward, the
    reference's BarrierRank, barrier.py:24-141) with the same kernels: the reference's
    `pipelined_over_barrier_wall` (harness.py:376-379)."""
    import torch
    import torch.distributed as dist

    def run(deferred):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            if deferred:
                bind.deferred = []
            step(dev_x, dev_y)  # step() calls bind.step_done(); flush before it counts the step
            if deferred:
                bind.k -= 1
                bind.flush()
                bind.k += 1
                bind.deferred = None
        bind.drain()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    run(False)  # warm both schedules
    run(True)
    p_ms, b_ms = run(False), run(True)
    return {"pipelined_ms_per_step": p_ms, "barrier_ms_per_step": b_ms, "pipelined_over_barrier_wall": p_ms / b_ms,
            "barrier_schedule": "same kernels, every layer exchanged after the full backward (eager steps)"}


def comparison_arm(args):
    """Comparison rows only: the phase-separated bulk schedule (full backward,
    one NCCL all-reduce of the flat gradient, then the libpgx fused update kernel), and
    PyTorch DDP (bucketed NCCL all-reduce overlapped with backward) + fused torch SGD."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1706_00095_b200 import _lib

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("cpu:gloo,cuda:nccl", rank=rank, world_size=world, device_id=dev)
    torch.backends.cudnn.benchmark = True
    wl = wl_of(args)
    model = wl["cls"]().to(dev)
    h = wl["hyper"]
    B = global_batch(wl, world) // world
    gb = B * world
    IMG = wl["image"]
    g = torch.Generator().manual_seed(42 + rank)
    dev_x = torch.randint(0, 256, (B, wl.get("channels", 3), IMG, IMG), dtype=torch.uint8, generator=g).to(dev)
    dev_y = torch.randint(0, wl.get("classes", 1000), (B,), dtype=torch.int64, generator=g).to(dev)
    params = [p for _, ps in model.layers() for p in ps]
    n = sum(p.numel() for p in params)
    if args.variant == "ddp":
        net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], gradient_as_bucket_view=True)
        opt = torch.optim.SGD(params, lr=h["lr"], momentum=h["momentum"], weight_decay=h["weight_decay"],
                              fused=True)
    else:
        net = model
        flat_w = torch.empty(n, device=dev)
        flat_g = torch.zeros(n, device=dev)
        flat_v = torch.zeros(n, device=dev)
        off = 0
        with torch.no_grad():
            for p in params:
                flat_w[off:off + p.numel()].copy_(p.reshape(-1))
                p.data = flat_w[off:off + p.numel()].view_as(p)
                p.grad = flat_g[off:off + p.numel()].view_as(p)
                off += p.numel()
        dist.broadcast(flat_w, 0)

    def step():
        xin = dev_x.to(torch.bfloat16, memory_format=torch.channels_last).sub_(128.0).mul_(1.0 / 64.0)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = net(xin)
        loss = model.loss(out, dev_y)
        if args.variant == "ddp":
            opt.zero_grad(set_to_none=False)
            loss.backward()
            opt.step()
        else:
            flat_g.zero_()
            loss.backward()
            dist.all_reduce(flat_g)  # bulk: one NCCL all-reduce after the whole backward
            parts = (C.c_void_p * 1)(flat_g.data_ptr())
            _lib.call("pgx_fold_update", _lib.MODE_FAST32, parts, 1, flat_w.data_ptr(), flat_v.data_ptr(), n,
                      h["lr"], 1.0 / world, h["momentum"], h["weight_decay"],
                      torch.cuda.current_stream().cuda_stream)
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=dist.new_group(backend="gloo"))
    ms = float(t.item())
    if rank == 0:
        cfg = workload_config(world, args)
        cfg["comparison"] = {"nccl_bulk": "phase-separated: backward, NCCL all-reduce of the flat gradient, "
                                          "libpgx fused update (barrier.py schedule)",
                             "ddp": "torch DDP bucketed NCCL all-reduce + fused torch SGD"}[args.variant]
        print(json.dumps({"metric": wl["metric"], "value": gb * args.steps / (ms / 1e3), "unit": "images/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": wl["scaling"],
                          "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg,
                          "impl": "comparison-" + args.variant}), flush=True)
    dist.destroy_process_group()


def ncu_traffic(kernel: str, world: int, layer_params: int):
    """(dram read+write bytes, NVLink tx bytes, source) per launch of the dominant kernel from
    the committed ncu captures (profiles/ncu_traffic.json) for this kernel/world/layer; None
    entries where no capture exists.  N=2 entries come from a run across two GPUs (NVLink
    counters included); 4 ranks stepped on one GPU are only a fallback (local peer stores)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            table = json.load(fh)
    except Exception:  # noqa: BLE001
        return None, None, None
    for key in (f"{kernel}/N{world}/{layer_params}", f"{kernel}/N{world}stepped/{layer_params}"):
        rec = table.get(key)
        if rec is not None:
            return rec["dram_read_bytes"] + rec["dram_write_bytes"], rec.get("nvltx_bytes"), \
                "profiles/ncu_traffic.json " + key
    return None, None, None


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback B200_PROFILING.md 6.65 TB/s"


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    elif args.variant in ("nccl_bulk", "ddp"):
        comparison_arm(args)
    else:
        pgx_arm(args)


if __name__ == "__main__":
    main()
