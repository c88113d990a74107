"""Device-timed C2 (BASELINE configs[1]: 256 pairs, L=256, d=8, lambda=2, RBF
sigma=1) forward and backward (dev tool)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402

kind = int(sys.argv[1]) if len(sys.argv) > 1 and __name__ == "__main__" else 1
rng = np.random.default_rng(0)


def paths(n, L, d):
    return torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1), device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


if __name__ == "__main__":
    x, y = paths(256, 256, 8), paths(256, 256, 8)
    tf = timed(lambda: ops.forward_batch(x, y, 2, 2, kind, 1.0))
    tb = timed(lambda: ops.backward_batch(x, y, 2, 2, kind, 1.0, None, want_values=True))
    print(f"C2 kind={kind}: fwd {tf:.3f} ms, bwd {tb:.3f} ms, total {tf + tb:.3f} ms")
