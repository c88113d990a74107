"""BASELINE config 2 (RBF, lambda 2) batch backward once, for ncu."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402
rng = np.random.default_rng(0)
def paths(n, L, d):
    return torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1), device="cuda")
x, y = paths(256, 256, 8), paths(256, 256, 8)
ops.backward_batch(x, y, 2, 2, 1, 1.0, None, want_values=True)
torch.cuda.synchronize()
