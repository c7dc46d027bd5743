"""Dense tanh MLP on the device with per-layer gradient emission (reference net.py).

The forward/backward stays plain PyTorch (it is not the path); what matters for
the path is the emission contract of backward_from_cache (net.py:163-172,
207-214): `on_layer(l, g_l)` fires in strictly decreasing l after layer l's
flat gradient [dW row-major][db] is final and after d_a was propagated through
W_l, so the callback may overwrite the weights of layers >= l.
"""

from __future__ import annotations

import torch

from .config import DenseLayerSpec, specs_from_dims  # noqa: F401  (re-export)
from .errors import InputError, ShapeError
from .ops import seeded_fill

_TAG_INPUTS = 0x696E70757473   # net.py:21
_TAG_TEACHER = 0x7465616368    # net.py:22


def _derived_seed(seed: int, *tags: int) -> int:
    m = (1 << 64) - 1

    def mix(z):
        z &= m
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)

    s = seed & m
    for t in tags:
        s = mix(s ^ mix(t & m))
    return s


derived_seed = _derived_seed


def split_params(spec: DenseLayerSpec, flat: torch.Tensor):
    if flat.numel() != spec.param_count:
        raise ShapeError(f"layer buffer has {flat.numel()} values, spec needs {spec.param_count}")
    n = spec.in_dim * spec.out_dim
    return flat[:n].view(spec.out_dim, spec.in_dim), flat[n:]


def init_model(seed: int, specs, dtype=torch.float64, device="cuda") -> list:
    """Layer l = seeded_fill(seed ^ l, S_l, 1/sqrt(in_dim)) (net.py:66-76)."""
    import math
    return [seeded_fill(seed ^ l, s.param_count, 1.0 / math.sqrt(s.in_dim), dtype, device) for l, s in enumerate(specs)]


class Dataset:
    def __init__(self, inputs: torch.Tensor, targets: torch.Tensor):
        if inputs.dim() != 2 or targets.dim() != 2:
            raise ShapeError("dataset inputs and targets must be 2-D")
        if inputs.shape[0] != targets.shape[0]:
            raise ShapeError(f"inputs hold {inputs.shape[0]} rows but targets hold {targets.shape[0]}")
        if inputs.shape[0] == 0:
            raise InputError("dataset must contain at least one sample")
        self.inputs, self.targets = inputs, targets

    def __len__(self) -> int:
        return self.inputs.shape[0]

    def take(self, idx):
        idx = torch.as_tensor(idx, device=self.inputs.device)
        return self.inputs[idx], self.targets[idx]


def forward(specs, weights, x):
    a = x
    cache = [a]
    for spec, flat in zip(specs, weights):
        w, b = split_params(spec, flat)
        z = torch.addmm(b, a, w.t())
        a = torch.tanh(z) if spec.activation == "tanh" else z
        cache.append(a)
    return a, cache


def batch_loss(out, t) -> torch.Tensor:
    d = out - t
    return (d * d).sum() / (2.0 * out.shape[1] * out.shape[0])


def backward_from_cache(specs, weights, cache, t, on_layer=None):
    """Per-layer gradients, output layer first (net.py:180-215)."""
    loss = batch_loss(cache[-1], t)
    n_out, b = specs[-1].out_dim, cache[0].shape[0]
    d_a = (cache[-1] - t) / (n_out * b)
    grads = [None] * len(specs)
    for l in range(len(specs) - 1, -1, -1):
        spec = specs[l]
        a_in, a_out = cache[l], cache[l + 1]
        d_z = d_a * (1.0 - a_out * a_out) if spec.activation == "tanh" else d_a
        w, _ = split_params(spec, weights[l])
        d_w = d_z.t() @ a_in
        d_b = d_z.sum(dim=0)
        d_a = d_z @ w  # propagate before emitting (net.py:207-210)
        g = torch.cat([d_w.reshape(-1), d_b])
        grads[l] = g
        if on_layer is not None:
            on_layer(l, g)
    return grads, loss


def backward(specs, weights, x, t, on_layer=None):
    if x.shape[0] == 0:
        raise InputError("batch must contain at least one sample")
    _, cache = forward(specs, weights, x)
    return backward_from_cache(specs, weights, cache, t, on_layer)


def make_synthetic_dataset(seed: int, num_samples: int, specs, input_scale: float = 1.0,
                           dtype=torch.float64, device="cuda") -> Dataset:
    """Seeded inputs + teacher-network targets (net.py:226-247); inputs are
    bit-identical to the reference's, targets come from the device forward."""
    if num_samples < 1:
        raise InputError(f"num_samples must be >= 1, got {num_samples}")
    flat = seeded_fill(_derived_seed(seed, _TAG_INPUTS), num_samples * specs[0].in_dim, input_scale, dtype, device)
    x = flat.view(num_samples, specs[0].in_dim)
    teacher = init_model(_derived_seed(seed, _TAG_TEACHER), specs, dtype, device)
    y, _ = forward(specs, teacher, x)
    return Dataset(x, y)
