"""Truncated signatures: device time of the forward and backward at the paper's
Table 1 shapes ((B, L, d, N) = (128, 256, 4, 6),
(128, 512, 8, 5), (128, 1024, 16, 4)), beside the C oracle (restatement of the
reference, all host threads) on a bounded sample.  Inputs: the reference bench
generator (bench.py:53-56), seed 0."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import signatures as sg  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def make_paths(rng, batch, length, dim):
    steps = rng.standard_normal((batch, length, dim)) / np.sqrt(max(length, 1))
    return np.cumsum(steps, axis=1, dtype=np.float64)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


out = {}
threads = os.cpu_count() or 1
for B, L, d, N in ((128, 256, 4, 6), (128, 512, 8, 5), (128, 1024, 16, 4)):
    rng = np.random.default_rng(0)
    X = make_paths(rng, B, L, d)
    x = torch.as_tensor(X, device="cuda")
    total = sum(d ** k for k in range(1, N + 1))
    cot = torch.as_tensor(rng.standard_normal((B, total)), device="cuda")
    tf = timed(lambda: sg.signature_forward(x, N))
    tb = timed(lambda: sg.signature_backward_t(x, N, cot), reps=1)
    # CPU oracle on a sample of paths (per-path cost is uniform)
    bs = 8
    t0 = time.perf_counter()
    orc.signature(X[:bs], N, threads=threads)
    cf = (time.perf_counter() - t0) * B / bs
    t0 = time.perf_counter()
    orc.signature_backward(X[:bs], N, cot[:bs].cpu().numpy(), threads=threads)
    cb = (time.perf_counter() - t0) * B / bs
    out[f"({B},{L},{d},{N})"] = {"gpu_fwd_s": tf, "gpu_bwd_s": tb, "cpu_port_fwd_s": cf,
                                 "cpu_port_bwd_s": cb, "cpu_threads": threads,
                                 "cpu_sample": f"{bs} of {B} paths, scaled"}
    print(f"({B},{L},{d},{N}): fwd {tf*1e3:.3f} ms, bwd {tb*1e3:.3f} ms; "
          f"CPU port fwd {cf:.3f} s, bwd {cb:.3f} s ({threads} threads)", flush=True)
print(json.dumps(out))
