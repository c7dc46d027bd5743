"""Benchmark networks (BASELINE.json configs): Caffe-prototxt-shaped PyTorch modules.

The networks are not the path — their forward/backward stays plain PyTorch — they
exist to drive the per-layer exchange with the reference configurations' layer
sizes and emission orders.  Every module exposes ``layers()`` -> [(module, [W, b])]
in model order: one exchange "layer" = one Caffe parameter layer, flattened
[W row-major][b] (the reference layer layout, net.py:57-63).
"""

from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F


class LRN(nn.Module):
    """Caffe/AlexNet across-channel LRN, the same function as nn.LocalResponseNorm:
    x / (k + alpha/size * sum_{c-size/2..c+size/2} x^2)^beta.  The channel window is summed
    with one avg_pool1d over the innermost dim of the channels-last activation (one kernel
    instead of pad + avg_pool3d + elementwise), in fp32; measured 12 % faster AlexNet steps
    (profiles/r1fb_fwdbwd_variants.jsonl) with identical results."""

    def __init__(self, size=5, alpha=1e-4, beta=0.75, k=1.0):
        super().__init__()
        self.size, self.alpha, self.beta, self.k = size, alpha, beta, k

    def forward(self, x):
        n, c, h, w = x.shape
        xl = x.permute(0, 2, 3, 1)
        xf = xl.float()
        s = F.avg_pool1d((xf * xf).reshape(-1, 1, c), self.size, stride=1, padding=self.size // 2,
                         count_include_pad=True)
        div = (s.reshape(n, h, w, c) * self.alpha + self.k).pow(self.beta)
        return (xf / div).to(x.dtype).permute(0, 3, 1, 2)


class AlexNet(nn.Module):
    """BVLC AlexNet (grouped conv2/4/5, LRN), 227x227: 60,965,224 params."""

    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 96, 11, stride=4)
        self.conv2 = nn.Conv2d(96, 256, 5, padding=2, groups=2)
        self.conv3 = nn.Conv2d(256, 384, 3, padding=1)
        self.conv4 = nn.Conv2d(384, 384, 3, padding=1, groups=2)
        self.conv5 = nn.Conv2d(384, 256, 3, padding=1, groups=2)
        self.fc6 = nn.Linear(9216, 4096)
        self.fc7 = nn.Linear(4096, 4096)
        self.fc8 = nn.Linear(4096, 1000)
        self.relu = nn.ReLU(inplace=True)
        self.lrn = LRN(5, alpha=1e-4, beta=0.75)
        self.pool = nn.MaxPool2d(3, 2)
        self.drop = nn.Dropout(0.5)

    def forward(self, x):
        x = self.pool(self.lrn(self.relu(self.conv1(x))))
        x = self.pool(self.lrn(self.relu(self.conv2(x))))
        x = self.relu(self.conv3(x))
        x = self.relu(self.conv4(x))
        x = self.pool(self.relu(self.conv5(x)))
        x = x.flatten(1)
        x = self.drop(self.relu(self.fc6(x)))
        x = self.drop(self.relu(self.fc7(x)))
        return self.fc8(x)

    def loss(self, out, y):
        return nn.functional.cross_entropy(out.float(), y)

    def layers(self):
        return [(m, [m.weight, m.bias]) for m in (self.conv1, self.conv2, self.conv3, self.conv4, self.conv5,
                                                 self.fc6, self.fc7, self.fc8)]


class _Inception(nn.Module):
    def __init__(self, cin, c1, c3r, c3, c5r, c5, cp):
        super().__init__()
        self.b1 = nn.Conv2d(cin, c1, 1)
        self.b3r = nn.Conv2d(cin, c3r, 1)
        self.b3 = nn.Conv2d(c3r, c3, 3, padding=1)
        self.b5r = nn.Conv2d(cin, c5r, 1)
        self.b5 = nn.Conv2d(c5r, c5, 5, padding=2)
        self.pp = nn.Conv2d(cin, cp, 1)

    def forward(self, x):
        r = torch.relu
        return torch.cat([r(self.b1(x)), r(self.b3(r(self.b3r(x)))), r(self.b5(r(self.b5r(x)))),
                          r(self.pp(nn.functional.max_pool2d(x, 3, 1, 1)))], 1)

    def convs(self):
        return [self.b1, self.b3r, self.b3, self.b5r, self.b5, self.pp]


class _Aux(nn.Module):
    def __init__(self, cin):
        super().__init__()
        self.conv = nn.Conv2d(cin, 128, 1)
        self.fc1 = nn.Linear(2048, 1024)
        self.fc2 = nn.Linear(1024, 1000)

    def forward(self, x):
        x = torch.relu(self.conv(nn.functional.avg_pool2d(x, 5, 3)))
        x = nn.functional.dropout(torch.relu(self.fc1(x.flatten(1))), 0.7, self.training)
        return self.fc2(x)


class GoogLeNet(nn.Module):
    """BVLC GoogLeNet with both auxiliary heads, 224x224: 64 parameter layers,
    13,378,280 params, many small layers."""

    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 64, 7, 2, 3)
        self.conv2r = nn.Conv2d(64, 64, 1)
        self.conv2 = nn.Conv2d(64, 192, 3, padding=1)
        self.lrn = LRN(5, alpha=1e-4, beta=0.75)
        self.i3a = _Inception(192, 64, 96, 128, 16, 32, 32)
        self.i3b = _Inception(256, 128, 128, 192, 32, 96, 64)
        self.i4a = _Inception(480, 192, 96, 208, 16, 48, 64)
        self.i4b = _Inception(512, 160, 112, 224, 24, 64, 64)
        self.i4c = _Inception(512, 128, 128, 256, 24, 64, 64)
        self.i4d = _Inception(512, 112, 144, 288, 32, 64, 64)
        self.i4e = _Inception(528, 256, 160, 320, 32, 128, 128)
        self.i5a = _Inception(832, 256, 160, 320, 32, 128, 128)
        self.i5b = _Inception(832, 384, 192, 384, 48, 128, 128)
        self.aux1 = _Aux(512)
        self.aux2 = _Aux(528)
        self.fc = nn.Linear(1024, 1000)

    def forward(self, x):
        mp = lambda t: nn.functional.max_pool2d(t, 3, 2, ceil_mode=True)  # noqa: E731
        x = self.lrn(mp(torch.relu(self.conv1(x))))
        x = mp(self.lrn(torch.relu(self.conv2(torch.relu(self.conv2r(x))))))
        x = mp(self.i3b(self.i3a(x)))
        x = self.i4a(x)
        a1 = self.aux1(x) if self.training else None
        x = self.i4d(self.i4c(self.i4b(x)))
        a2 = self.aux2(x) if self.training else None
        x = mp(self.i4e(x))
        x = self.i5b(self.i5a(x))
        x = nn.functional.dropout(nn.functional.adaptive_avg_pool2d(x, 1).flatten(1), 0.4, self.training)
        return self.fc(x), a1, a2

    def loss(self, out, y):
        main, a1, a2 = out
        ce = nn.functional.cross_entropy
        l = ce(main.float(), y)
        if a1 is not None:
            l = l + 0.3 * (ce(a1.float(), y) + ce(a2.float(), y))
        return l

    def layers(self):
        mods = [self.conv1, self.conv2r, self.conv2]
        for blk in (self.i3a, self.i3b, self.i4a, self.i4b, self.i4c, self.i4d, self.i4e, self.i5a, self.i5b):
            mods += blk.convs()
        mods += [self.aux1.conv, self.aux1.fc1, self.aux1.fc2, self.aux2.conv, self.aux2.fc1, self.aux2.fc2, self.fc]
        return [(m, [m.weight, m.bias]) for m in mods]


class LeNet(nn.Module):
    """Caffe lenet_train_test.prototxt (configs[0], the CPU reference's own workload shape):
    520 / 25,050 / 400,500 / 5,010 params."""

    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(1, 20, 5)
        self.conv2 = nn.Conv2d(20, 50, 5)
        self.ip1 = nn.Linear(800, 500)
        self.ip2 = nn.Linear(500, 10)

    def forward(self, x):
        x = F.max_pool2d(self.conv1(x), 2, 2)
        x = F.max_pool2d(self.conv2(x), 2, 2)
        return self.ip2(torch.relu(self.ip1(x.flatten(1))))

    def loss(self, out, y):
        return F.cross_entropy(out.float(), y)

    def layers(self):
        return [(m, [m.weight, m.bias]) for m in (self.conv1, self.conv2, self.ip1, self.ip2)]


class Cifar10Quick(nn.Module):
    """Caffe cifar10_quick (configs[1]): 2,432 / 25,632 / 51,264 / 65,600 / 650 params."""

    def __init__(self):
        super().__init__()
        self.conv1 = nn.Conv2d(3, 32, 5, padding=2)
        self.conv2 = nn.Conv2d(32, 32, 5, padding=2)
        self.conv3 = nn.Conv2d(32, 64, 5, padding=2)
        self.ip1 = nn.Linear(1024, 64)
        self.ip2 = nn.Linear(64, 10)

    def forward(self, x):
        x = torch.relu(F.max_pool2d(self.conv1(x), 3, 2, ceil_mode=True))
        x = F.avg_pool2d(torch.relu(self.conv2(x)), 3, 2, ceil_mode=True)
        x = F.avg_pool2d(torch.relu(self.conv3(x)), 3, 2, ceil_mode=True)
        return self.ip2(self.ip1(x.flatten(1)))

    def loss(self, out, y):
        return F.cross_entropy(out.float(), y)

    def layers(self):
        return [(m, [m.weight, m.bias]) for m in (self.conv1, self.conv2, self.conv3, self.ip1, self.ip2)]


WORKLOADS = {
    "alexnet": dict(cls=AlexNet, image=227, global_batch=256, scaling="strong",
                    hyper=dict(lr=0.01, momentum=0.9, weight_decay=5e-4),
                    metric="AlexNet images/sec (B=256 global, synthetic 227x227), per-layer gradient exchange"),
    "googlenet": dict(cls=GoogLeNet, image=224, per_gpu_batch=32, scaling="weak",
                      hyper=dict(lr=0.01, momentum=0.9, weight_decay=2e-4),
                      metric="GoogLeNet images/sec (B=32 per GPU, synthetic 224x224), per-layer gradient exchange"),
    "lenet": dict(cls=LeNet, image=28, channels=1, classes=10, global_batch=64, scaling="strong",
                  hyper=dict(lr=0.01, momentum=0.0, weight_decay=0.0), reference_world=2,
                  metric="LeNet-5 images/sec (B=64 global, synthetic 28x28), per-layer gradient exchange"),
    "cifar10_quick": dict(cls=Cifar10Quick, image=32, classes=10, per_gpu_batch=100, scaling="weak",
                          hyper=dict(lr=0.001, momentum=0.9, weight_decay=0.004), reference_world=4,
                          metric="cifar10_quick images/sec (B=100 per GPU, synthetic 32x32), per-layer gradient "
                                 "exchange"),
}
