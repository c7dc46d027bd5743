"""Benchmark networks: Caffe layer sizes and the LRN formulation."""

import torch

import workloads as W


def test_alexnet_and_googlenet_layer_sizes():
    a = [sum(p.numel() for p in ps) for _, ps in W.AlexNet().layers()]
    assert a == [34944, 307456, 885120, 663936, 442624, 37752832, 16781312, 4097000]
    g = [sum(p.numel() for p in ps) for _, ps in W.GoogLeNet().layers()]
    assert len(g) == 64 and sum(g) == 13378280


def test_lrn_matches_torch_local_response_norm():
    torch.manual_seed(0)
    x = torch.randn(2, 96, 9, 9).contiguous(memory_format=torch.channels_last) * 3
    ref = torch.nn.LocalResponseNorm(5, alpha=1e-4, beta=0.75)(x)
    got = W.LRN(5, alpha=1e-4, beta=0.75)(x)
    torch.testing.assert_close(got, ref, rtol=1e-6, atol=1e-6)
    x2 = torch.randn(2, 7, 5, 5) * 10  # NCHW input and a channel count below the window
    torch.testing.assert_close(W.LRN()(x2), torch.nn.LocalResponseNorm(5, 1e-4, 0.75)(x2), rtol=1e-6, atol=1e-6)
