"""Split the small-call cost (BASELINE configs[0]) into: the raw C-ABI call
(ctypes, plan, prep + solve launches), ops.forward_batch, sig_kernel (dev tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2509_10613_b200 as sk  # noqa: E402
from paper_2509_10613_b200 import _lib, ops  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
x = torch.as_tensor(bench.make_paths(rng, 32, 64, 4), device=dev)
y = torch.as_tensor(bench.make_paths(rng, 32, 64, 4), device=dev)
lib = _lib.load()
out = torch.empty(32, dtype=torch.float64, device=dev)
nb = lib.sk_forward_batch_tf_workspace_bytes(32, 64, 64, 4, 0, 0, 0, 0)
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
args = (x.data_ptr(), y.data_ptr(), 32, 64, 64, 4, 0, 0, 0, 1.0, 0, out.data_ptr(),
        ws.data_ptr(), nb, st)


def per_call(fn, n=3000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print(f"empty ctypes call (sk_abi_version): {per_call(lambda: lib.sk_abi_version()):.2f} us")
print(f"workspace query (ctypes):           {per_call(lambda: lib.sk_forward_batch_tf_workspace_bytes(32, 64, 64, 4, 0, 0, 0, 0)):.2f} us")
print(f"raw C ABI launch call:              {per_call(lambda: lib.sk_forward_batch_tf(*args)):.2f} us")
print(f"ops.forward_batch:                  {per_call(lambda: ops.forward_batch(x, y, 0, 0, 0, 1.0)):.2f} us")
print(f"sig_kernel:                         {per_call(lambda: sk.sig_kernel(x, y)):.2f} us")
print(f"torch.empty(32):                    {per_call(lambda: torch.empty(32, dtype=torch.float64, device=dev)):.2f} us")

# the same call captured once in a CUDA graph and replayed (inputs copied into
# the captured buffers): the small-call path without host-side launch work
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        sk.sig_kernel(x, y)
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    kg = sk.sig_kernel(x, y)
print(f"sig_kernel as a CUDA-graph replay:  {per_call(lambda: graph.replay()):.2f} us")
