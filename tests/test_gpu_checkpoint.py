"""PSGD1 checkpoints packed / unpacked by the device kernels (pgx_ckpt_pack/unpack)
against the reference's own bytes (golden) and the oracle restatement at full AlexNet
size.  Parity bar: bit-exact bytes."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle import pipesgd_oracle as O

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "formats_golden.npz"))
M = json.load(open(os.path.join(HERE, "golden", "formats_golden.json")))
LENET = [520, 25050, 400500, 5010]
ALEXNET = [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]


def small_layers():
    return [G[f"ckpt_small_l{i}"] for i in range(4)]


def test_serialize_matches_reference_bytes():
    from paper_1706_00095_b200.checkpoint import serialize_model

    dev = [torch.from_numpy(a.copy()).cuda() for a in small_layers()]
    assert serialize_model(dev) == G["ckpt_small_blob"].tobytes()


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_serialize_lenet_sha(dt):
    from paper_1706_00095_b200.checkpoint import serialize_model

    w = [O.seeded_fill(42 ^ l, n, 1.0 / np.sqrt(n)) for l, n in enumerate(LENET)]
    if dt == "f32":
        w = [a.astype(np.float32) for a in w]
    blob = serialize_model([torch.from_numpy(a).cuda() for a in w])
    assert hashlib.sha256(blob).hexdigest() == M[f"ckpt_lenet_{dt}_sha256"]


def test_load_reference_blob_bitwise():
    from paper_1706_00095_b200.checkpoint import load_model_bytes

    m = load_model_bytes(G["ckpt_small_blob"].tobytes())
    assert m.iteration == 0
    for got, want in zip(m.layers, small_layers()):
        assert got.dtype == torch.float64
        assert got.cpu().numpy().view(np.uint64).tobytes() == want.view(np.uint64).tobytes()
    m32 = load_model_bytes(G["ckpt_small_blob"].tobytes(), dtype=torch.float32)
    for got, want in zip(m32.layers, small_layers()):
        w32 = want.astype(np.float32)
        g = got.cpu().numpy()
        nan = np.isnan(w32)
        assert np.array_equal(np.isnan(g), nan)
        assert g[~nan].view(np.uint32).tobytes() == w32[~nan].view(np.uint32).tobytes()


@pytest.mark.parametrize("case", sorted(M["ckpt_errors"]))
def test_load_errors(case):
    from paper_1706_00095_b200.checkpoint import load_model_bytes
    from paper_1706_00095_b200.errors import FormatError

    with pytest.raises(FormatError) as ei:
        load_model_bytes(G[f"ckpt_bad_{case}"].tobytes())
    assert str(ei.value) == M["ckpt_errors"][case]


@pytest.mark.parametrize("sizes", [[0, 1, 5, 0, 3], [1], [7, 0], ALEXNET, [(i * 7) % 34 for i in range(700)]])
def test_ragged_and_full_size_roundtrip(sizes, tmp_path):
    """Ragged / empty layers, the full AlexNet model (fp32 as the exchange holds it) and a
    700-layer model (more layers than the kernel-parameter table holds: the table goes
    through device memory; the format has no layer limit): bytes equal the oracle's image,
    and loading them back is the identity."""
    from paper_1706_00095_b200.checkpoint import load_model, save_model

    g = torch.Generator(device="cuda").manual_seed(1706)
    layers = [torch.randn(n, generator=g, device="cuda") for n in sizes]
    path = str(tmp_path / "m.psgd")
    save_model(layers, path)
    host = [t.cpu().numpy() for t in layers]
    blob = open(path, "rb").read()
    assert hashlib.sha256(blob).digest() == hashlib.sha256(O.ckpt_serialize(host)).digest()
    back = load_model(path, dtype=torch.float32)
    for a, b in zip(back.layers, layers):
        assert torch.equal(a, b)


def test_exchange_checkpoint_roundtrip(tmp_path):
    from paper_1706_00095_b200.checkpoint import load_exchange, save_exchange
    from paper_1706_00095_b200.exchange import DeviceExchange
    from paper_1706_00095_b200.transport import LocalWorld

    world = LocalWorld(1, inline=False)
    tr = world.transport(0)
    x = DeviceExchange(tr, LENET, mode="fast32", variant="twoshot", lr=0.01)
    x.connect()
    for l, n in enumerate(LENET):
        x.layer_views[l].copy_(torch.from_numpy(O.seeded_fill(42 ^ l, n, 0.1).astype(np.float32)))
    path = str(tmp_path / "x.psgd")
    save_exchange(x, path)
    saved = [v.clone() for v in x.layer_views]
    for v in x.layer_views:
        v.zero_()
    load_exchange(x, path)
    for a, b in zip(x.layer_views, saved):
        assert torch.equal(a, b)
    assert O.ckpt_load(open(path, "rb").read())[2].tobytes() == saved[2].cpu().double().numpy().tobytes()
    x.close()
    tr.close()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_pack_unpack_on_a_non_current_device():
    """Layers on cuda:1 while cuda:0 is current: the kernels must launch on the layers' device."""
    from paper_1706_00095_b200.checkpoint import load_model_bytes, serialize_model

    torch.cuda.set_device(0)
    dev = [torch.from_numpy(a.copy()).to("cuda:1") for a in small_layers()]
    blob = serialize_model(dev)
    assert blob == G["ckpt_small_blob"].tobytes()
    back = load_model_bytes(blob, device="cuda:1")
    for a, t in zip(small_layers(), back.layers):
        assert t.device.index == 1 and t.cpu().numpy().tobytes() == a.astype(np.float64).tobytes()
