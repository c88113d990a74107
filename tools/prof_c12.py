"""BASELINE configs 1 and 2 once each (for ncu): C1 forward (linear, 32 pairs,
L 64, d 4), C2 forward and backward (RBF sigma 1, lambda 2, 256 pairs, L 256, d 8)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402

rng = np.random.default_rng(0)


def paths(n, L, d):
    return torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1),
                           device="cuda")


x1, y1 = paths(32, 64, 4), paths(32, 64, 4)
ops.forward_batch(x1, y1, 0, 0, 0, 1.0)
x, y = paths(256, 256, 8), paths(256, 256, 8)
ops.forward_batch(x, y, 2, 2, 1, 1.0)
ops.backward_batch(x, y, 2, 2, 1, 1.0, None, want_values=True)
torch.cuda.synchronize()
