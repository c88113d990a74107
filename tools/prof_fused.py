"""One fused value + gradient Gram pass at a given size (ncu capture driver):
prof_fused.py [n] [L] [d]  (default: the bench's C3 shape)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2509_10613_b200 as sk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
L = int(sys.argv[2]) if len(sys.argv) > 2 else 512
d = int(sys.argv[3]) if len(sys.argv) > 3 else 16
rng = np.random.default_rng(0)
X = torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1), device="cuda")
G, g, _ = sk.sig_kernel_gram_value_and_grad(X)
torch.cuda.synchronize()
print("ok", float(G[0, 0]), float(g.abs().max()))
