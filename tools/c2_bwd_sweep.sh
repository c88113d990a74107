#!/bin/bash
# C2 backward (RBF / linear, lambda 2, 256 pairs, L 256, d 8) device time per forced NW
for nw in 1 4 8; do
  SK_BWD_XW_NW=$nw python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2509_10613_b200 import ops
rng = np.random.default_rng(0)
p = lambda n, L, d: torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / 16, 1), device='cuda')
x, y = p(256, 256, 8), p(256, 256, 8)
cases = (('C2 rbf', lambda: ops.backward_batch(x, y, 2, 2, 1, 1.0, None, want_values=True)),
         ('C2 linear', lambda: ops.backward_batch(x, y, 2, 2, 0, 1.0, None, want_values=True)))
for name, fn in cases:
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): fn()
    b.record(); torch.cuda.synchronize()
    print(f"NW={os.environ['SK_BWD_XW_NW']} {name} bwd: {a.elapsed_time(b)/3:.3f} ms", flush=True)
PY
done
