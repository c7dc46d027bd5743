"""Isolated launches of the dominant kernel (fc6 exchange/update, k_twoshot) for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1706_00095_b200.exchange import DeviceExchange
from paper_1706_00095_b200.transport import DistTransport

L = [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]
tr = DistTransport(0, 1, 0)
x = DeviceExchange(tr, L, mode="fast32", lr=0.01, momentum=0.9, weight_decay=5e-4,
                   chunk_elems=int(os.environ.get("CHUNK", "16384")), max_ctas=int(os.environ.get("CTAS", "0")))
tr.barrier(); x.connect()
g = [torch.randn(4096, 9216, device="cuda") * 1e-3, torch.randn(4096, device="cuda") * 1e-3]
ts = []
for i in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(x.stream); x.launch(5, i, g); e1.record(x.stream); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
nvl, hbm = x.layer_bytes(5)
print("fc6 launch ms", ts, "GB/s", [hbm / (t / 1e3) / 1e9 for t in ts])
x.close(); tr.close()
