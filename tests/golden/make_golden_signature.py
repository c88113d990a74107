"""Golden fixtures for the truncated-signature path, made by running the
REFERENCE (sigcore signature / signature_backward, signature.py:104-121,
signature_grad.py:20-53).  Run in the build container only:

    cd /tmp && NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_golden_signature.py
"""

import os

import numpy as np

import sigcore as sc  # the reference, via PYTHONPATH

OUT = os.path.dirname(os.path.abspath(__file__))
TF = {None: 0, "time_augment": 1, "lead_lag": 2}


def random_paths(rng, b, length, d, scale=1.0):
    """reference tests/conftest.py:24-27."""
    steps = rng.standard_normal((b, length, d)) / np.sqrt(max(length - 1, 1))
    return np.cumsum(steps, axis=1) * scale


CASES = [  # (B, L, d, depth, transform, custom times, repeated points)
    (3, 12, 2, 4, None, False, False),
    (2, 9, 3, 5, "time_augment", False, False),
    (2, 7, 2, 3, "lead_lag", False, False),
    (1, 20, 4, 3, "time_augment", True, False),
    (2, 6, 1, 6, None, False, False),
    (4, 32, 4, 6, None, False, False),
    (2, 10, 8, 3, None, False, False),
    (2, 8, 16, 2, "lead_lag", False, False),
    (2, 9, 2, 4, None, False, True),
    (1, 40, 2, 10, None, False, False),
]


def main():
    rng = np.random.default_rng(2024)
    arrays = {"n": np.array(len(CASES))}
    for i, (B, L, d, depth, kind, custom, rep) in enumerate(CASES):
        x = random_paths(rng, B, L, d)
        if rep:
            x[:, 3] = x[:, 2]  # zero increment inside the path (the skipped step)
            x[:, -1] = x[:, -2]
        times = np.sort(rng.uniform(0, 1, L)) if custom else None
        if custom:
            times[0], times[-1] = 0.0, 1.0
        opts = sc.SigOptions(depth, transform=kind)
        pb = sc.PathBatch(x, times=times)
        sig = sc.signature(pb, opts)
        cot = rng.standard_normal(sig.shape)
        grad = sc.signature_backward(pb, opts, cot)
        arrays.update({f"s{i}_x": x, f"s{i}_sig": sig, f"s{i}_cot": cot, f"s{i}_grad": grad,
                       f"s{i}_meta": np.array([depth, TF[kind], int(custom)]),
                       f"s{i}_times": times if custom else np.zeros(0)})
    path = os.path.join(OUT, "signature.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


if __name__ == "__main__":
    main()
