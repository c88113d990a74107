"""Device time of batch forward / backward at a few training-like shapes (dev tool)."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2509_10613_b200 import ops  # noqa: E402
from time_c2 import paths, timed  # noqa: E402

for B, L, d, lam, kind in ((4096, 128, 8, 0, 0), (1024, 256, 16, 0, 0), (4096, 64, 4, 1, 1),
                           (512, 512, 8, 1, 0), (2048, 128, 32, 0, 0)):
    x, y = paths(B, L, d), paths(B, L, d)
    tf = timed(lambda: ops.forward_batch(x, y, lam, lam, kind, 1.0), 5)
    tb = timed(lambda: ops.backward_batch(x, y, lam, lam, kind, 1.0, None, want_values=True), 3)
    cells = B * ((L - 1) << lam) ** 2
    print(f"B={B} L={L} d={d} lam={lam} kind={kind}: fwd {tf:.3f} ms ({cells / tf / 1e9:.2f} Gcell/ms), "
          f"bwd {tb:.3f} ms ({cells / tb / 1e9:.2f} Gcell/ms)")
