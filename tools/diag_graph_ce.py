"""Diagnose device-iteration (graph) mode across 2 GPUs: one layer, eager iterations,
then a captured launch+gate replayed; prints the flag words after every replay."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1706_00095_b200.exchange import DeviceExchange
from paper_1706_00095_b200.transport import DistTransport

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
variant = sys.argv[1] if len(sys.argv) > 1 else "twoshot_ce"
tr = DistTransport(rank, world, rank, timeout_s=5.0)
x = DeviceExchange(tr, [1 << 16], mode="fast32", variant=variant, lr=0.01)
tr.barrier(); x.connect()
g = torch.ones(1 << 16, device="cuda")
mseg, rseg = tr.segment(16), tr.segment(17)
def flags():
    torch.cuda.synchronize()
    return tr.notify_poll(16, 0, mseg.notification_count), tr.notify_poll(17, 0, rseg.notification_count)
for k in range(3):
    x.launch(0, k, [g]); x.gate(0, k, stream=x.stream)
torch.cuda.synchronize(); dist.barrier()
print(rank, "eager flags", flags(), "status", tr.device_status(), flush=True)
x.set_device_iteration(True, 2)
graph = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream(); cap.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cap), torch.cuda.graph(graph, stream=cap):
    x.tick(cap)
    x.gate(0, -1, stream=cap)
    x.stream.wait_stream(cap)
    x.launch(0, 0, [g])
    x.join(0, cap)
torch.cuda.current_stream().wait_stream(cap); torch.cuda.synchronize(); dist.barrier()
for r in range(3):
    t0 = time.time(); graph.replay(); torch.cuda.synchronize()
    print(rank, "replay", r, "%.3fs" % (time.time() - t0), flags(), "status", tr.device_status(), flush=True)
    dist.barrier()
x.close(); tr.close()
