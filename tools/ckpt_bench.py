"""PSGD1 checkpoint kernels at AlexNet size (fp32 model, 60,965,224 params): pack and
unpack launch times (CUDA events) against measured HBM bandwidth, and save/load
end to end.  Algorithmic bytes: pack reads 4n and writes 8n (+12 per layer + 5);
unpack reads the 8n image and writes 4n."""
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1706_00095_b200 import _lib  # noqa: E402
from paper_1706_00095_b200.checkpoint import load_model, pack, save_model, unpack_into, serialize_model  # noqa: E402
import ctypes as C  # noqa: E402

ALEXNET = [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]
n = sum(ALEXNET)
g = torch.Generator(device="cuda").manual_seed(0)
layers = [torch.randn(k, generator=g, device="cuda") for k in ALEXNET]
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6544.3


def timeit(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(300 * 1965)  # hide the host's enqueue: the events bracket device time
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


img, nbytes = pack(layers)
t_pack = timeit(lambda: pack(layers, out=img))
blob = serialize_model(layers)
out = [torch.empty_like(t) for t in layers]
words = (nbytes + 7) // 8 + 1
dimg = torch.zeros(words * 8, dtype=torch.uint8, device="cuda")
dimg[:nbytes].copy_(torch.frombuffer(bytearray(blob), dtype=torch.uint8))
ptrs = (C.c_void_p * len(out))(*[t.data_ptr() for t in out])
cnt = (C.c_uint64 * len(out))(*ALEXNET)


def unpack():
    _lib.call("pgx_ckpt_unpack", C.c_void_p(dimg.data_ptr()), words * 8, cnt, len(out), 4, ptrs,
              C.c_void_p(torch.cuda.current_stream().cuda_stream))


t_unpack = timeit(unpack)
assert all(torch.equal(a, b) for a, b in zip(out, layers))
path = "/tmp/alexnet.psgd"
t0 = time.perf_counter()
save_model(layers, path)
t_save = time.perf_counter() - t0
t0 = time.perf_counter()
m = load_model(path, dtype=torch.float32)
torch.cuda.synchronize()
t_load = time.perf_counter() - t0
assert all(torch.equal(a, b) for a, b in zip(m.layers, layers))
pb = 4 * n + nbytes
ub = nbytes + 4 * n
print(json.dumps({"what": "PSGD1 checkpoint of the AlexNet fp32 model", "params": n, "image_bytes": nbytes,
                  "pack_ms": t_pack, "pack_GBps": pb / t_pack / 1e6, "pack_frac_hbm": pb / t_pack / 1e6 / peak,
                  "unpack_ms": t_unpack, "unpack_GBps": ub / t_unpack / 1e6, "unpack_frac_hbm": ub / t_unpack / 1e6 / peak,
                  "hbm_peak_GBps": peak, "save_model_s": t_save, "load_model_s": t_load,
                  "note": "pack/unpack: one kernel each, CUDA events, median of 20; save/load: wall clock incl. "
                          "D2H/H2D and file IO"}))
