"""FP32-arithmetic vs fp64 fused Gram value + gradient at the C3 shape (and
the C5 shape on a sub-Gram): device time with CUDA events, and the error of a
sub-block against the fp64 kernels (python tools/time_f32_bwd.py [n])."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_10613_b200 as sk  # noqa: E402


def brownian(rng, n, L, d):
    return np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return min(ts)


out = {}
for name, n, L, d in [("C3 1024^2 L512 d16", int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 512, 16),
                      ("C5-shape 2048^2 L1024 d8", 2048, 1024, 8)]:
    rng = np.random.default_rng(0)
    X = torch.as_tensor(brownian(rng, n, L, d), device="cuda")
    X32 = X.float()
    C = torch.ones((n, n), dtype=torch.float64, device="cuda")
    t64 = timed(lambda: sk.sig_kernel_gram_value_and_grad(X, None, C))
    t32 = timed(lambda: sk.sig_kernel_gram_value_and_grad(X32, None, C, precision="fp32"))
    G64, g64, _ = sk.sig_kernel_gram_value_and_grad(X32.double(), None, C)
    G32, g32, _ = sk.sig_kernel_gram_value_and_grad(X32, None, C, precision="fp32")
    cells = n * (n + 1) / 2 * (L - 1) ** 2
    out[name] = {
        "fp64_s": t64, "fp32_s": t32, "speedup": t64 / t32,
        "fp32_cells_per_s": cells / t32,
        "G_rel_err": float((G32.double() - G64).abs().max() / G64.abs().max()),
        "grad_rel_err": float((g32.double() - g64).abs().max() / g64.abs().max()),
    }
    print(name, out[name], flush=True)
print(json.dumps(out))
