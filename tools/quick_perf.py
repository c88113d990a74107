"""Quick device-timed forward throughput on the BASELINE shapes (dev tool)."""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2509_10613_b200 as sk  # noqa: E402
from paper_2509_10613_b200 import ops  # noqa: E402


def paths(n, L, d, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.cumsum(torch.randn(n, L, d, generator=g, device="cuda", dtype=torch.float64)
                        / L ** 0.5, dim=1)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


res = {}
# C3 forward (Gram 1024^2, L=512, d=16)
X = paths(1024, 512, 16)
t = timeit(lambda: ops.forward_gram(X, None, 0, 0, 0, 1.0))
cells = 1024 * 1025 / 2 * 511 ** 2
res["c3_fwd"] = {"s": t, "cells_per_s": cells / t, "dp_instr_per_s": cells / t * 23}
# C5-shaped sub Gram 2048^2, L=1024, d=8
X5 = paths(2048, 1024, 8)
t = timeit(lambda: ops.forward_gram(X5, None, 0, 0, 0, 1.0), reps=1)
cells = 2048 * 2049 / 2 * 1023 ** 2
res["c5sub_fwd"] = {"s": t, "cells_per_s": cells / t, "dp_instr_per_s": cells / t * 15}
# C4 forward (B=128, L=8192, d=4, lam=1)
x4, y4 = paths(128, 8192, 4, 1), paths(128, 8192, 4, 2)
t = timeit(lambda: ops.forward_batch(x4, y4, 1, 1, 0, 1.0), reps=2)
cells = 128 * 16382 ** 2
res["c4_fwd"] = {"s": t, "cells_per_s": cells / t, "dp_instr_per_s": cells / t * 5}
# C2 forward RBF (B=256, L=256, d=8, lam=2)
x2, y2 = paths(256, 256, 8, 3), paths(256, 256, 8, 4)
t = timeit(lambda: ops.forward_batch(x2, y2, 2, 2, 1, 1.0))
cells = 256 * 1020 ** 2
res["c2_fwd_rbf"] = {"s": t, "cells_per_s": cells / t}
print(json.dumps(res, indent=1))
