"""A/B of two library builds on the C3 fused G + gradient (run once per build
with SK_LIBSIGKERNEL set): device time over 3 reps and the outputs saved for a
bitwise comparison.  python tools/ab_c3.py <tag> [n]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_10613_b200 as sk  # noqa: E402

tag = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rng = np.random.default_rng(0)
X = torch.as_tensor(np.cumsum(rng.standard_normal((n, 512, 16)) / np.sqrt(512), axis=1), device="cuda")
C = torch.as_tensor(rng.standard_normal((n, n)), device="cuda")
res = {}
for name, xx, prec in [("fp64", X, "fp64"), ("fp32", X.float(), "fp32")]:
    out = sk.sig_kernel_gram_value_and_grad(xx, None, C, precision=prec)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        s.record()
        out = sk.sig_kernel_gram_value_and_grad(xx, None, C, precision=prec)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    res[name] = (min(ts), out[0].cpu(), out[1].cpu())
    print(f"{tag} {name}: {min(ts):.1f} ms", flush=True)
torch.save(res, f"gpurun_out/ab_{tag}.pt")
