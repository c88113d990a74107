#!/bin/bash
# C2 forward (RBF / linear, lambda 2, 256 pairs, L 256, d 8) device time per forced XW width
for w in 0 2 4 8 16; do
  SK_FWD_XW_W=$w python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_10613_b200 import ops
rng = np.random.default_rng(0)
p = lambda n, L, d: torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / 16, 1), device='cuda')
x, y = p(256, 256, 8), p(256, 256, 8)
x4, y4 = p(128, 8192, 4), p(128, 8192, 4)
cases = (('C2 rbf', lambda: ops.forward_batch(x, y, 2, 2, 1, 1.0)),
         ('C2 linear', lambda: ops.forward_batch(x, y, 2, 2, 0, 1.0)),
         ('C4 linear', lambda: ops.forward_batch(x4, y4, 1, 1, 0, 1.0)))
for name, fn in cases:
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): fn()
    b.record(); torch.cuda.synchronize()
    print(f"W={os.environ['SK_FWD_XW_W']} {name} fwd: {a.elapsed_time(b)/5:.3f} ms")
PY
done
