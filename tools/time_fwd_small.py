"""Device time per call of small / Gram forwards on the r01 FMA-pipe kernels
(C1 batch, a dyadic-order Gram, an RBF Gram) -- dev tool."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402
from time_c2 import paths, timed  # noqa: E402

x, y = paths(32, 64, 4), paths(32, 64, 4)
print(f"C1 fwd: {timed(lambda: ops.forward_batch(x, y, 0, 0, 0, 1.0), 200) * 1e3:.2f} us")
X = paths(256, 128, 8)
print(f"Gram 256 L128 d8 lam1 fwd: {timed(lambda: ops.forward_gram(X, None, 1, 1, 0, 1.0), 5):.3f} ms")
print(f"Gram 256 L128 d8 RBF fwd: {timed(lambda: ops.forward_gram(X, None, 0, 0, 1, 1.0), 5):.3f} ms")
x2, y2 = paths(4096, 128, 8), paths(4096, 128, 8)
print(f"batch 4096 L128 d8 fwd: {timed(lambda: ops.forward_batch(x2, y2, 0, 0, 0, 1.0), 5):.3f} ms")
xr, yr = paths(4096, 128, 8), paths(4096, 128, 8)
print(f"batch 4096 L128 d8 RBF lam1 fwd: {timed(lambda: ops.forward_batch(xr, yr, 1, 1, 1, 1.0), 5):.3f} ms")
Xr = paths(512, 64, 4)
print(f"Gram 512 L64 d4 RBF lam2 fwd: {timed(lambda: ops.forward_gram(Xr, None, 2, 2, 1, 1.0), 5):.3f} ms")
