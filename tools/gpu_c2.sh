mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_backward_gpu.py tests/test_forward_gpu.py tests/test_conformance_gpu.py -q -x > gpurun_out/c2_tests.log 2>&1; echo "rc $?" >> gpurun_out/c2_tests.log
timeout 600 python - > gpurun_out/c2.log 2>&1 <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2509_10613_b200 import ops
rng = np.random.default_rng(0)
def paths(n, L, d): return torch.as_tensor(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L), axis=1), device="cuda")
x, y = paths(256, 256, 8), paths(256, 256, 8)
f = lambda: ops.backward_batch(x, y, 2, 2, 1, 1.0, None, want_values=True)
f(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); [f() for _ in range(5)]; b.record(); torch.cuda.synchronize()
print("C2 bwd ms", a.elapsed_time(b) / 5)
PY
