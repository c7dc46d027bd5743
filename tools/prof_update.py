"""Isolated launches of the dominant kernel (fc6 exchange/update at N=1, k_twoshot<1>): device
time per launch (a ~100 us busy kernel queued ahead of the start event hides the host enqueue)
for a list of chunk sizes / CTA caps, and as an ncu target.

    python tools/prof_update.py [CHUNK:CTAS ...]      (default 16384:0 = bench.py's plan)
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
from paper_1706_00095_b200.exchange import DeviceExchange
from paper_1706_00095_b200.transport import DistTransport

L = [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]
PEAK = 6548.2  # MEASURED_PEAKS.json hbm_gbs on this pool
tr = DistTransport(0, 1, 0)
g = [torch.randn(4096, 9216, device="cuda") * 1e-3, torch.randn(4096, device="cuda") * 1e-3]
configs = sys.argv[1:] or ["16384:0"]
for cfg in configs:
    chunk, ctas = (int(v) for v in cfg.split(":"))
    x = DeviceExchange(tr, L, mode="fast32", lr=0.01, momentum=0.9, weight_decay=5e-4, seg_base=16 + 4 * configs.index(cfg),
                       chunk_elems=chunk, max_ctas=ctas)
    tr.barrier()
    x.connect()
    ts = []
    for i in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(x.stream):
            torch.cuda._sleep(200000)
        e0.record(x.stream)
        x.launch(5, i, g)
        e1.record(x.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[5:])
    nvl, hbm = x.layer_bytes(5)
    med = ts[len(ts) // 2]
    print(json.dumps({"chunk": chunk, "ctas": ctas, "plan": x.layer_plan(5), "median_ms": med, "min_ms": ts[0],
                      "gbs": hbm / (med / 1e3) / 1e9, "frac": hbm / (med / 1e3) / 1e9 / PEAK}), flush=True)
    x.close()
tr.close()
