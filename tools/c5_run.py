"""One full BASELINE config 5 step on one GPU: symmetric sig_kernel_gram of
8192 Brownian paths (L=1024, d=8, lambda=0), fp64 G + gradient (cotangent
ones; argv[2] = "fused" (default, one value+grad pass) or "split"), device-timed, with a sub-block parity check against the C
oracle.  Writes a JSON summary (evidence run; bench.py's default is C3)."""
import json
import sys
import time

import numpy as np
import torch

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
from paper_2509_10613_b200 import ops  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
L, d = 1024, 8
rng = np.random.default_rng(0)
X = np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1)
Xd = torch.as_tensor(X, device="cuda")
C = torch.ones((n, n), dtype=torch.float64, device="cuda")
peak = ops.dfma_peak()
torch.cuda.synchronize()
mode = sys.argv[2] if len(sys.argv) > 2 else "fused"
pairs = n * (n + 1) // 2
cells = pairs * (L - 1) ** 2
t0 = time.time()
if mode == "fused":
    # one value + gradient pass (sig_kernel_gram_value_and_grad's kernel call)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    G, gx, _ = ops.value_and_grad_gram(Xd, None, 0, 0, 0, 1.0, C)
    e[1].record()
    torch.cuda.synchronize()
    step_s = e[0].elapsed_time(e[1]) / 1e3
    out = {"config": f"C5 sym Gram n={n} L={L} d={d} lambda=0 fp64 G + gradient (fused value+grad "
                     f"pass), cotangent ones, 1 GPU",
           "step_s": step_s, "wall_s": time.time() - t0,
           "cells": cells, "cells_per_s": cells / step_s, "gram_entries_per_s": n * n / step_s,
           "step_frac_of_dfma_algorithmic": cells * 40 / step_s / peak,
           "executed_frac_of_dfma": cells * (27 + 4 * d) / step_s / peak,
           "dfma_peak_fma_per_s": peak}
else:
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    G = ops.forward_gram(Xd, None, 0, 0, 0, 1.0)
    e[1].record()
    gx, _ = ops.backward_gram(Xd, None, 0, 0, 0, 1.0, C)
    e[2].record()
    torch.cuda.synchronize()
    fwd_s = e[0].elapsed_time(e[1]) / 1e3
    bwd_s = e[1].elapsed_time(e[2]) / 1e3
    out = {"config": f"C5 sym Gram n={n} L={L} d={d} lambda=0 fp64 fwd+bwd, cotangent ones, 1 GPU",
           "fwd_s": fwd_s, "bwd_s": bwd_s, "step_s": fwd_s + bwd_s, "wall_s": time.time() - t0,
           "cells": cells, "cells_per_s": cells / (fwd_s + bwd_s),
           "gram_entries_per_s": n * n / (fwd_s + bwd_s),
           "fwd_frac_of_dfma": cells * 15 / fwd_s / peak,
           "bwd_frac_of_dfma_algorithmic": cells * 25 / bwd_s / peak,
           "step_frac_of_dfma_algorithmic": cells * 40 / (fwd_s + bwd_s) / peak,
           "dfma_peak_fma_per_s": peak}
# parity of a sub-block (first 6 paths) and symmetry
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402  (checker only)
Gs = G[:6, :6].cpu().numpy()
want = orc.kernel_gram(X[:6])
out["subblock_rel_err"] = float(np.abs(Gs - want).max() / np.abs(want).max())
out["symmetric_exact"] = bool(torch.equal(G, G.T))
out["grad_finite"] = bool(torch.isfinite(gx).all().item())
out["grad_abs_max"] = float(gx.abs().max().item())
# full-size parity of one Gram row and one path's gradient: G[0, :] is k(x_0, x_b)
# over all n paths, and with cotangent ones dF/dx_0 = 2 sum_b d1 k(x_0, x_b)
# (k(x, y) = k(y, x): the column-side terms equal the row-side ones), i.e. the
# cross Gram backward of x_0 against every path with cotangent 2 -- n pairs of
# the full L = 1024 grid on the CPU oracle (all host threads)
t1 = time.time()
row = orc.kernel_gram(X[:1], X, 0, 0)
out["row0_rel_err"] = float(np.abs(G[0].cpu().numpy() - row[0]).max() / np.abs(row[0]).max())
g0, _ = orc.gram_backward(X[:1], X, 2.0 * np.ones((1, n)), 0, 0)
got0 = gx[0].cpu().numpy()
out["grad_path0_rel_err"] = float(np.abs(got0 - g0[0]).max() / np.abs(g0[0]).max())
out["oracle_check_s"] = time.time() - t1
out["oracle_check"] = (f"G[:6,:6], G[0,:] ({n} pairs) and dF/dx_0 ({n} pairs, cross Gram backward "
                       f"with cotangent 2) vs oracle/sk_oracle.c; tolerance 1e-10")
print(json.dumps(out, indent=1))
