"""Full-size parity evidence against the C oracle (all host threads):
C3 -- the whole 1024 x 1024 Gram G of the fused value + gradient step and the
gradient of path 0 (1024-pair cross Gram backward, cotangent 2: with cotangent
ones dF/dx_0 = 2 sum_b d1 k(x_0, x_b) by symmetry); C4 -- all 128 pairs of the
forward at L = 8192.  Inputs: the reference bench generator, seed 0.  Writes
one JSON object (evidence run; the -m gpu tests use sub-blocks)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
import paper_2509_10613_b200 as sk  # noqa: E402
from oracle import oracle as orc  # noqa: E402  (checker only)


def make_paths(rng, b, L, d):
    return np.cumsum(rng.standard_normal((b, L, d)) / np.sqrt(L), axis=1)


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


out = {"oracle_threads": os.cpu_count()}
# C3
rng = np.random.default_rng(0)
X = make_paths(rng, 1024, 512, 16)
ones = torch.ones((1024, 1024), dtype=torch.float64, device="cuda")
G, gx, _ = sk.sig_kernel_gram_value_and_grad(torch.as_tensor(X, device="cuda"), None, ones)
G, gx = G.cpu().numpy(), gx.cpu().numpy()
t0 = time.time()
Gw = orc.kernel_gram(X, None, 0, 0)
g0, _ = orc.gram_backward(X[:1], X, 2.0 * np.ones((1, 1024)), 0, 0)
out["C3"] = {"what": "full 1024^2 G (525,312 pairs) and dF/dx_0 of the fused step vs the oracle",
             "G_rel_err": rel(G, Gw), "G_symmetric_exact": bool((G == G.T).all()),
             "grad_path0_rel_err": rel(gx[0], g0[0]), "oracle_s": time.time() - t0}
# C4
rng = np.random.default_rng(0)
x = make_paths(rng, 128, 8192, 4)
y = make_paths(rng, 128, 8192, 4)
k = sk.sig_kernel(torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda"),
                  dyadic_order=1).cpu().numpy()
t0 = time.time()
kw = orc.kernel_batch(x, y, 1, 1)
out["C4"] = {"what": "all 128 pairs, L=8192, d=4, lambda=1 forward vs the oracle",
             "rel_err": rel(k, kw), "oracle_s": time.time() - t0}
out["tolerance"] = 1e-10
print(json.dumps(out, indent=1))
