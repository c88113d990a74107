"""Device-timed C4 (BASELINE configs[3]: 128 pairs, L=8192, d=4, lambda=1,
linear) forward (dev tool)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402
from time_c2 import paths, timed  # noqa: E402

x, y = paths(128, 8192, 4), paths(128, 8192, 4)
t = timed(lambda: ops.forward_batch(x, y, 1, 1, 0, 1.0), 5)
print(f"C4 fwd {t:.3f} ms, {128 * 16382 ** 2 / t * 1e3:.3e} cells/s")
