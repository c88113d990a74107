"""Per-call latency of the small-problem path (BASELINE config 1: 32 pairs,
L=64, d=4, lambda=0): host wall time per call (async enqueue, averaged over
many calls, one sync at the end) and device time per call."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_10613_b200 as sk  # noqa: E402
from paper_2509_10613_b200 import ops  # noqa: E402


def main(n=2000):
    rng = np.random.default_rng(0)
    x = torch.as_tensor(np.cumsum(rng.standard_normal((32, 64, 4)) / 8, 1), device="cuda")
    y = torch.as_tensor(np.cumsum(rng.standard_normal((32, 64, 4)) / 8, 1), device="cuda")
    res = {}
    for name, fn in (("ops.forward_batch", lambda: ops.forward_batch(x, y, 0, 0, 0, 1.0)),
                     ("sig_kernel", lambda: sk.sig_kernel(x, y))):
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / n * 1e6
        dev = e0.elapsed_time(e1) / n * 1e3
        res[name] = (wall, dev)
        print(f"{name}: {wall:.2f} us/call host, {dev:.2f} us/call device stream")
    # one blocking call end to end (enqueue + kernel + sync)
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        sk.sig_kernel(x, y)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"sig_kernel blocking: median {np.median(ts) * 1e6:.2f} us")
    return res


if __name__ == "__main__":
    main()
