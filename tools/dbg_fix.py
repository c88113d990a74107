import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2509_10613_b200 import ops, gram_dist
def random_paths(rng, b, length, d, scale=1.0):
    steps = rng.standard_normal((b, length, d)) / np.sqrt(max(length - 1, 1))
    return np.cumsum(steps, axis=1) * scale
rng = np.random.default_rng(22)
X = random_paths(rng, 19, 45, 8)
x = torch.as_tensor(X, device='cuda')
C = torch.ones((19, 19), dtype=torch.float64, device='cuda')
for rg in [(0, 19), (16, 19), (0, 8), (8, 16)]:
    acc = ops.GradAcc(19, 45, 8, x.device).init(C, 19, 19, True)
    ops.value_and_grad_gram(x, None, 0, 0, 0, 1.0, C, rows=rg, acc_x=acc)
    m = acc.meta.cpu().numpy()
    g = acc.finalize()
    print(rg, 'meta', m[:4], 'maxc', np.frombuffer(m[0:1].tobytes(), np.float64), 'nscale', np.frombuffer(m[2:3].tobytes(), np.float64), 'finite', bool(torch.isfinite(g).all()))
    out, gx, _ = ops.value_and_grad_gram(x, None, 0, 0, 0, 1.0, C, rows=rg)
    print('   plain finite', bool(torch.isfinite(gx).all()), float(gx.abs().max()))
