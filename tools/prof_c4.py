"""BASELINE config 4 (128 pairs, L=8192, d=4, lambda=1, linear) forward once,
for ncu captures."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402

rng = np.random.default_rng(0)
x, y = (torch.as_tensor(np.cumsum(rng.standard_normal((128, 8192, 4)) / np.sqrt(8192), axis=1),
                        device="cuda") for _ in range(2))
ops.forward_batch(x, y, 1, 1, 0, 1.0)
torch.cuda.synchronize()
