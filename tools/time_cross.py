"""Cross Gram with the longer paths on the y side: the whole-Gram call (solved
as G^T on the DMMA tiles) against the same call with an explicit full row
range (the forward keeps the swapped orientation, FMA-pipe kernels; the
backward is transposed either way), and the difference between the two.  python tools/time_cross.py [n] [Lx] [Ly] [d]"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402

n, Lx, Ly, d = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (256, 256, 384, 16)))
rng = np.random.default_rng(0)
X = torch.as_tensor(np.cumsum(rng.standard_normal((n, Lx, d)) / np.sqrt(Lx), axis=1), device="cuda")
Y = torch.as_tensor(np.cumsum(rng.standard_normal((n, Ly, d)) / np.sqrt(Ly), axis=1), device="cuda")
C = torch.as_tensor(rng.standard_normal((n, n)), device="cuda")


def timed(fn, reps=3):
    r = fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, r


for name, kw in (("whole (G^T on DMMA)", {}), ("row range (swapped, FMA pipe)", {"rows": (0, n)})):
    tf, G = timed(lambda: ops.forward_gram(X, Y, 0, 0, 0, 1.0, **kw))
    tb, R = timed(lambda: ops.value_and_grad_gram(X, Y, 0, 0, 0, 1.0, C, **kw))
    print(f"{name}: forward {tf:.1f} ms, value+grad {tb:.1f} ms", flush=True)
    if not kw:
        ref = (G, R)
print("G bitwise equal:", torch.equal(ref[0], G), " value+grad G bitwise:", torch.equal(ref[1][0], R[0]))
for i in (1, 2):
    e = (ref[1][i] - R[i]).abs().max() / R[i].abs().max()
    print(f"gradient {i} rel diff {e.item():.2e}")
