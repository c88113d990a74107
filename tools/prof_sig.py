"""Truncated-signature backward at (B, L, d, N) = (128, 512, 8, 5), once, for ncu."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import signatures as sg  # noqa: E402
B, L, d, N = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (128, 512, 8, 5)))
rng = np.random.default_rng(0)
X = np.cumsum(rng.standard_normal((B, L, d)) / np.sqrt(L), axis=1)
x = torch.as_tensor(X, device="cuda")
total = sum(d ** k for k in range(1, N + 1))
cot = torch.as_tensor(rng.standard_normal((B, total)), device="cuda")
sg.signature_backward_t(x, N, cot)
torch.cuda.synchronize()
