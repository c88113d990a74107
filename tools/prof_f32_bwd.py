"""fp64 then FP32-arithmetic fused Gram value + gradient at the C3 shape
(n paths) for ncu captures of both gram_bwd_mma instances."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2509_10613_b200 as sk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
rng = np.random.default_rng(0)
X = torch.as_tensor(np.cumsum(rng.standard_normal((n, 512, 16)) / np.sqrt(512), axis=1),
                    device="cuda")
C = torch.ones((n, n), dtype=torch.float64, device="cuda")
sk.sig_kernel_gram_value_and_grad(X, None, C)
sk.sig_kernel_gram_value_and_grad(X.float(), None, C, precision="fp32")
torch.cuda.synchronize()
