"""Device-timed throughput of every BASELINE.json config on one GPU (evidence run).

C1 fwd, C2 fwd + bwd (RBF, sigma 1), C3 fused G + gradient, C4 fwd, C5 on a
2048-path sub-Gram (the full 8192^2 run is tools/c5_run.py).  Each line:
cells/s and the fraction of the live FP64 peak at the algorithmic DP count
(SURVEY.md 8d).  Inputs: the reference generator (_make_paths, seed 0)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2509_10613_b200 as sk  # noqa: E402
from paper_2509_10613_b200 import ops  # noqa: E402


def paths(rng, n, L, d):
    return torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1),
                           device="cuda")


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def dp(d, l1, l2):
    f = 2.0 ** (l1 + l2)
    return 3 + (d + 4) / f, 7 + (2 * d + 2) / f


peak = ops.dfma_peak()
rng = np.random.default_rng(0)
out = {"peak_fma_per_s": peak}

x, y = paths(rng, 32, 64, 4), paths(rng, 32, 64, 4)
t = timed(lambda: ops.forward_batch(x, y, 0, 0, 0, 1.0), 50)
c = 32 * 63 ** 2
out["C1 sig_kernel fwd B32 L64 d4 lam0"] = {"s": t, "cells_per_s": c / t,
                                            "frac": c * dp(4, 0, 0)[0] / t / peak}

x, y = paths(rng, 256, 256, 8), paths(rng, 256, 256, 8)
tf = timed(lambda: ops.forward_batch(x, y, 2, 2, 1, 1.0), 20)
tb = timed(lambda: ops.backward_batch(x, y, 2, 2, 1, 1.0, None, want_values=True), 5)
c = 256 * 1020 ** 2
out["C2 sig_kernel fwd+bwd B256 L256 d8 lam2 RBF"] = {
    "fwd_s": tf, "bwd_s": tb, "fwd_cells_per_s": c / tf, "bwd_cells_per_s": c / tb,
    "values_and_grad_one_call_s": tb,
    "one_call": "bwd_s is the backward WITH the values (want_values=True): the reference's "
                "kernel_batch_backward contract (kernel_grad.py:64-98), sig_kernel_value_and_grad",
    "note": "RBF adds an exp per coarse node; frac not reported (SURVEY 8d counts linear)"}

X = paths(rng, 1024, 512, 16)
ones = torch.ones((1024, 1024), dtype=torch.float64, device="cuda")
t = timed(lambda: sk.sig_kernel_gram_value_and_grad(X, None, ones), 2)
c = 1024 * 1025 // 2 * 511 ** 2
out["C3 Gram 1024^2 L512 d16 fused G+grad"] = {"s": t, "cells_per_s": c / t,
                                              "frac": c * sum(dp(16, 0, 0)) / t / peak}

x, y = paths(rng, 128, 8192, 4), paths(rng, 128, 8192, 4)
t = timed(lambda: ops.forward_batch(x, y, 1, 1, 0, 1.0), 5)
c = 128 * 16382 ** 2
out["C4 sig_kernel fwd B128 L8192 d4 lam1"] = {"s": t, "cells_per_s": c / t,
                                               "frac": c * dp(4, 1, 1)[0] / t / peak}

X = paths(rng, 2048, 1024, 8)
ones = torch.ones((2048, 2048), dtype=torch.float64, device="cuda")
t = timed(lambda: sk.sig_kernel_gram_value_and_grad(X, None, ones), 1)
c = 2048 * 2049 // 2 * 1023 ** 2
out["C5-shape sub-Gram 2048^2 L1024 d8 fused G+grad (full 8192^2: profiles/r01_c5_full_1gpu_fused.json)"] = {
    "s": t, "cells_per_s": c / t, "frac": c * sum(dp(8, 0, 0)) / t / peak}
# FP32-arithmetic forward kernels (precision='fp32', linear kernel) against the
# FP32 FMA pipe: 148 SMs x 128 lanes x 1.965 GHz (max SM clock) (FP32 instr/cell: the
# small-correction cell is 5 + (d + 4)/2^(l1+l2), sk_cell.cuh Coef32)
peak32 = 148 * 128 * 1.965e9
X32 = paths(rng, 1024, 512, 16).float()
t = timed(lambda: ops.forward_gram_f32(X32, None, 0, 0), 2)
c = 1024 * 1025 // 2 * 511 ** 2
out["C3-shape Gram fwd FP32 arithmetic"] = {"s": t, "cells_per_s": c / t,
                                            "frac_fp32": c * (5 + 20) / t / peak32,
                                            "peak_fp32_fma_per_s": peak32,
                                            "note": "float recurrence on the FMA pipe; p = <dx, dy> "
                                                    "on the FP64 tensor cores (DMMA), rounded "
                                                    "once to float -- frac_fp32 counts it as "
                                                    "FP32 work (d + 4 per cell)"}
ones = torch.ones((1024, 1024), dtype=torch.float64, device="cuda")
t = timed(lambda: sk.sig_kernel_gram_value_and_grad(X32, None, ones, precision="fp32"), 2)
out["C3 Gram fused G+grad FP32 arithmetic"] = {
    "s": t, "cells_per_s": c / t,
    "note": "float forward / recompute / small-correction adjoint on the FP32 pipe, p, gx, gy "
            "on the FP64 tensor cores (gram_bwd_mma<16,2,false,float>); same shape as C3"}
x, y = paths(rng, 128, 8192, 4).float(), paths(rng, 128, 8192, 4).float()
t = timed(lambda: ops.forward_batch_f32(x, y, 1, 1), 5)
c = 128 * 16382 ** 2
out["C4 sig_kernel fwd FP32 arithmetic"] = {"s": t, "cells_per_s": c / t,
                                            "frac_fp32": c * (5 + 8 / 4) / t / peak32}
import bench  # noqa: E402
out["C1 latency"] = bench.small_call_latency(torch.device("cuda", 0))
print(json.dumps(out, indent=1))
