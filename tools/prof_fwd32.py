"""FP32-arithmetic Gram forward timing: prof_fwd32.py n L d [lam]."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402

n, L, d = (int(a) for a in sys.argv[1:4])
lam = int(sys.argv[4]) if len(sys.argv) > 4 else 0
rng = np.random.default_rng(0)
X = torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1),
                    device="cuda").float()
ops.forward_gram_f32(X, None, lam, lam)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ops.forward_gram_f32(X, None, lam, lam)
e1.record()
torch.cuda.synchronize()
cells = n * (n + 1) / 2 * (((L - 1) << lam) ** 2)
ms = e0.elapsed_time(e1)
print(f"fp32 fwd n={n} L={L} d={d} lam={lam}: {ms:.2f} ms, {cells / ms * 1e3:.3e} cells/s")
