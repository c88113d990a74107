import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2509_10613_b200 as sk
from paper_2509_10613_b200 import ops
def random_paths(rng, b, length, d, scale=1.0):
    steps = rng.standard_normal((b, length, d)) / np.sqrt(max(length - 1, 1))
    return np.cumsum(steps, axis=1) * scale
rng = np.random.default_rng(22)
X = random_paths(rng, 19, 45, 8)
C = torch.ones((19, 19), dtype=torch.float64, device="cuda")
bad = 0
for i in range(30):
    x = torch.as_tensor(X, device='cuda')
    G, gx, _ = sk.sig_kernel_gram_value_and_grad(x, None, C)
    if not torch.isfinite(gx).all(): bad += 1
print('fused full: nan runs', bad, '/30')
for n in (7, 5, 19, 8, 9, 16, 17):
    X = random_paths(rng, n, 30, 8)
    cnt = 0
    for i in range(10):
        acc = ops.GradAcc(n, 30, 8, torch.device('cuda')).init(torch.ones((n, n), dtype=torch.float64, device='cuda'), n, n, True)
        ops.backward_gram(torch.as_tensor(X, device='cuda'), None, 0, 0, 0, 1.0, torch.ones((n, n), dtype=torch.float64, device='cuda'), acc_x=acc)
        if int(acc.meta[1]) != 0: cnt += 1
    print('n', n, 'flagged', cnt, '/10')
