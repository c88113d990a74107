"""cProfile of the small-call path (BASELINE configs[0] through sig_kernel):
where the host microseconds per call go (dev tool)."""
import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2509_10613_b200 as sk  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda", 0)
print(bench.small_call_latency(dev))
rng = np.random.default_rng(0)
x = torch.as_tensor(bench.make_paths(rng, 32, 64, 4), device=dev)
y = torch.as_tensor(bench.make_paths(rng, 32, 64, 4), device=dev)
for _ in range(100):
    sk.sig_kernel(x, y)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    sk.sig_kernel(x, y)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
