"""Device time of the Gram backward at a dyadic order: prof_bwd_dy.py n L d lam."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402

n, L, d, lam = (int(a) for a in sys.argv[1:5])
rng = np.random.default_rng(0)
X = torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1), device="cuda")
C = torch.ones((n, n), dtype=torch.float64, device="cuda")
ops.backward_gram(X, None, lam, lam, 0, 1.0, C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ops.backward_gram(X, None, lam, lam, 0, 1.0, C)
e1.record()
torch.cuda.synchronize()
print(f"bwd n={n} L={L} d={d} lam={lam}: {e0.elapsed_time(e1):.2f} ms")
