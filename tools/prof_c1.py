"""BASELINE config 1 forward (32 pairs, L=64, d=4) a few times, for ncu."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/", 1)[0])
import torch  # noqa: E402
from paper_2509_10613_b200 import ops  # noqa: E402
from time_c2 import paths  # noqa: E402
x, y = paths(32, 64, 4), paths(32, 64, 4)
for _ in range(3):
    ops.forward_batch(x, y, 0, 0, 0, 1.0)
torch.cuda.synchronize()
