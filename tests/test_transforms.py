"""Path transforms of the torch API against the reference (tests/golden/transforms.npz):
forward values and, through autograd, the reference's transform_adjoint."""

import numpy as np
import pytest
import torch

from conftest import golden, make_paths, rel_err
from paper_2509_10613_b200.api import path_transform


@pytest.mark.parametrize("kind,gkey,akey", [("time_augment", "g_ta", "adj_ta"),
                                            ("lead_lag", "g_ll", "adj_ll")])
def test_transform_and_adjoint_match_reference(kind, gkey, akey):
    g = golden("transforms")
    x = torch.as_tensor(g["x"]).requires_grad_(True)
    z = path_transform(x, kind)
    np.testing.assert_array_equal(z.detach().numpy(), g[kind])
    (z * torch.as_tensor(g[gkey])).sum().backward()
    np.testing.assert_allclose(x.grad.numpy(), g[akey], rtol=0, atol=1e-15)


@pytest.mark.gpu
def test_transformed_kernel_vs_oracle(oracle):
    import paper_2509_10613_b200 as sk
    g = golden("transforms")
    rng = np.random.default_rng(5)
    x = make_paths(rng, 3, 12, 2)
    y = make_paths(rng, 3, 9, 2)
    for kind in ("time_augment", "lead_lag"):
        xt = path_transform(torch.as_tensor(x), kind).numpy()
        yt = path_transform(torch.as_tensor(y), kind).numpy()
        want = oracle.kernel_batch(xt, yt, 1, 1)
        got = sk.sig_kernel(torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda"),
                            1, transform=kind).cpu().numpy()
        assert rel_err(got, want) < 1e-10
    X = torch.as_tensor(x, device="cuda").requires_grad_(True)
    assert torch.autograd.gradcheck(
        lambda a: sk.sig_kernel_gram(a, dyadic_order=0, transform="lead_lag"), (X,))
    del g
