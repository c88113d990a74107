"""Small C3-shaped Gram fwd+bwd for ncu captures (n=128 -> 8256 pairs)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
L = int(sys.argv[2]) if len(sys.argv) > 2 else 512
d = int(sys.argv[3]) if len(sys.argv) > 3 else 16
rng = np.random.default_rng(0)
X = torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1), device="cuda")
C = torch.ones((n, n), dtype=torch.float64, device="cuda")
for _ in range(2):
    ops.forward_gram(X, None, 0, 0, 0, 1.0)
    ops.backward_gram(X, None, 0, 0, 0, 1.0, C)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
ops.forward_gram(X, None, 0, 0, 0, 1.0)
e[1].record()
ops.backward_gram(X, None, 0, 0, 0, 1.0, C)
e[2].record()
torch.cuda.synchronize()
pairs = n * (n + 1) / 2
cells = pairs * (L - 1) ** 2
print(f"n={n} L={L} d={d}: fwd {e[0].elapsed_time(e[1]):.2f} ms ({cells / e[0].elapsed_time(e[1]) / 1e6:.3e} cells/s), "
      f"bwd {e[1].elapsed_time(e[2]):.2f} ms ({cells / e[1].elapsed_time(e[2]) / 1e6:.3e} cells/s)")
