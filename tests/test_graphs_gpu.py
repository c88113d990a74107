"""CUDA-graph capture of the public calls: the kernels launch on torch's
current stream with caller buffers and no synchronisation, so a call can be
captured once and replayed on new inputs copied into the captured buffers
(the small-call latency path: BASELINE config 1 as one graph replay)."""

import numpy as np
import pytest
import torch

from conftest import make_paths, rel_err

pytestmark = pytest.mark.gpu


def test_graph_replay_sig_kernel_and_gram():
    import paper_2509_10613_b200 as sk
    rng = np.random.default_rng(0)
    x = torch.as_tensor(make_paths(rng, 32, 64, 4), device="cuda")
    y = torch.as_tensor(make_paths(rng, 32, 64, 4), device="cuda")
    X = torch.as_tensor(make_paths(rng, 12, 40, 16), device="cuda")
    C = torch.as_tensor(rng.standard_normal((12, 12)), device="cuda")
    # warm up on a side stream (plans, workspaces), then capture
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            sk.sig_kernel(x, y)
            sk.sig_kernel_gram_value_and_grad(X, None, C)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        k = sk.sig_kernel(x, y)
        G, gx, _ = sk.sig_kernel_gram_value_and_grad(X, None, C)
    # new inputs into the captured buffers, replay, compare with eager calls
    x2 = torch.as_tensor(make_paths(rng, 32, 64, 4), device="cuda")
    X2 = torch.as_tensor(make_paths(rng, 12, 40, 16), device="cuda")
    x.copy_(x2)
    X.copy_(X2)
    g.replay()
    torch.cuda.synchronize()
    k_e = sk.sig_kernel(x2, y)
    G_e, gx_e, _ = sk.sig_kernel_gram_value_and_grad(X2, None, C)
    np.testing.assert_array_equal(k.cpu().numpy(), k_e.cpu().numpy())
    np.testing.assert_array_equal(G.cpu().numpy(), G_e.cpu().numpy())
    assert rel_err(gx.cpu().numpy(), gx_e.cpu().numpy()) == 0.0
