"""AlexNet forward+backward cost under equivalent formulations (compute only, no exchange):
LRN as nn.LocalResponseNorm vs a channels-last avg_pool1d window, conv1 input in NCHW vs
channels_last.  CUDA-graph captured steps, B in {256, 64, 32}."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn as nn
import torch.nn.functional as F
from workloads import AlexNet


class LRNWindow(nn.Module):
    """Same math as nn.LocalResponseNorm(size, alpha, beta, k): x / (k + alpha/size * sum_{window} x^2)^beta,
    the channel window summed with one avg_pool1d over the innermost (channels-last) dim."""

    def __init__(self, size=5, alpha=1e-4, beta=0.75, k=1.0):
        super().__init__()
        self.size, self.alpha, self.beta, self.k = size, alpha, beta, k

    def forward(self, x):
        n, c, h, w = x.shape
        xl = x.permute(0, 2, 3, 1)  # view: channels-last memory -> contiguous last dim
        sq = (xl.float() * xl.float()).reshape(-1, 1, c)
        s = F.avg_pool1d(sq, self.size, stride=1, padding=self.size // 2, count_include_pad=True)
        div = (s.reshape(n, h, w, c) * self.alpha + self.k).pow(self.beta)
        return (xl / div).to(x.dtype).permute(0, 3, 1, 2)


def build(lrn, conv1_nchw):
    m = AlexNet().cuda()
    if lrn == "window":
        m.lrn = LRNWindow()
    return m


# env: OPT=sgd|none (plain SGD step inside the graph or fwd+bwd alone), BATCHES=256,64,32,
# FAST=1 (only bench.py's formulation: torch LRN, channels-last conv1)
OPT = os.environ.get("OPT", "sgd")
BATCHES = [int(b) for b in os.environ.get("BATCHES", "256,64,32").split(",")]
LRNS = ("torch",) if os.environ.get("FAST") else ("torch", "window")
C1S = (False,) if os.environ.get("FAST") else (False, True)


def run(lrn, conv1_nchw, B, steps=20):
    torch.manual_seed(0)
    m = build(lrn, conv1_nchw)
    x = torch.randint(0, 256, (B, 3, 227, 227), dtype=torch.uint8, device="cuda")
    y = torch.randint(0, 1000, (B,), device="cuda")
    opt = torch.optim.SGD(m.parameters(), lr=0.01)

    def step():
        if conv1_nchw:
            xin = x.to(torch.bfloat16).sub_(128.0).mul_(1 / 64.0)
        else:
            xin = x.to(torch.bfloat16, memory_format=torch.channels_last).sub_(128.0).mul_(1 / 64.0)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            if conv1_nchw:
                h = m.conv1(xin).contiguous(memory_format=torch.channels_last)
                h = m.pool(m.lrn(m.relu(h)))
                h = m.pool(m.lrn(m.relu(m.conv2(h))))
                h = m.relu(m.conv3(h)); h = m.relu(m.conv4(h)); h = m.pool(m.relu(m.conv5(h)))
                h = h.flatten(1); h = m.drop(m.relu(m.fc6(h))); h = m.drop(m.relu(m.fc7(h))); out = m.fc8(h)
            else:
                out = m(xin)
        loss = F.cross_entropy(out.float(), y)
        loss.backward()
        if OPT == "sgd":
            opt.step()
        opt.zero_grad(set_to_none=False)
        return loss
    torch.backends.cudnn.benchmark = True
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


# numerics: the window LRN equals nn.LocalResponseNorm
t = torch.randn(4, 96, 27, 27, device="cuda").contiguous(memory_format=torch.channels_last)
ref = nn.LocalResponseNorm(5, alpha=1e-4, beta=0.75)(t)
got = LRNWindow()(t)
print(json.dumps({"lrn_max_rel_err": float(((got - ref).abs() / ref.abs().clamp_min(1e-6)).max())}))
for B in BATCHES:
    for lrn in LRNS:
        for c1 in C1S:
            print(json.dumps({"B": B, "lrn": lrn, "conv1_nchw": c1, "opt": OPT, "ms": run(lrn, c1, B)}), flush=True)
