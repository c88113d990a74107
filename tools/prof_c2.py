"""BASELINE config 2 (RBF sigma 1, lambda 2, 256 pairs, L=256, d=8) forward
and/or batch backward once, for ncu.  argv[1]: 'b' (backward, default), 'f'
(forward) or 'fb' (both)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402
what = sys.argv[1] if len(sys.argv) > 1 else "b"
rng = np.random.default_rng(0)
def paths(n, L, d):
    return torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1), device="cuda")
x, y = paths(256, 256, 8), paths(256, 256, 8)
if "f" in what:
    ops.forward_batch(x, y, 2, 2, 1, 1.0)
if "b" in what:
    ops.backward_batch(x, y, 2, 2, 1, 1.0, None, want_values=True)
torch.cuda.synchronize()
