"""GPU benchmark tasks in the reference's bench-report format.

The reference's harness (sigcore/bench.py:20-98; schema
schemas/bench_report.schema.json) times `kernel-fwd` / `kernel-bwd` on CPU
arrays: one warm-up, `reps` repetitions, the minimum wall time.  This module
runs the same tasks on the B200 kernels, plus Gram tasks, and reports in the
same fields; the extensions (device timing, solved PDE cells/s, roofline
fraction against a live FP64 peak) are described by
schemas/bench_report_gpu.schema.json.

Timing: inputs are generated as the reference does (`_make_paths`: cumulative
sums of N(0, 1/L) steps, seed 0), moved to the GPU outside the clock, and each
repetition is timed with CUDA events around the library call (device time).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidArgument

TASKS = ("kernel-fwd", "kernel-bwd", "gram-fwd", "gram-bwd", "gram-value-grad")


@dataclass
class BenchReport:
    """One run: the reference's fields (task, shape, repetitions, times,
    minimum, threads, scalar_width) plus GPU extensions."""

    task: str
    shape: dict
    repetitions: int
    times: list
    minimum: float = field(init=False)
    threads: int = 1
    scalar_width: int = 64
    device: str = "cuda"
    timing: str = "cuda-events"
    cells: int = 0
    cells_per_s: float = 0.0
    roofline_frac: float | None = None

    def __post_init__(self):
        self.minimum = min(self.times)
        self.cells_per_s = self.cells / self.minimum if self.minimum > 0 else 0.0

    def to_dict(self) -> dict:
        return {"task": self.task, "shape": self.shape, "repetitions": self.repetitions,
                "times": self.times, "minimum": self.minimum, "threads": self.threads,
                "scalar_width": self.scalar_width, "device": self.device,
                "timing": self.timing, "cells": self.cells, "cells_per_s": self.cells_per_s,
                "roofline_frac": self.roofline_frac}

    def to_json(self, indent=None) -> str:
        return json.dumps(self.to_dict(), indent=indent)


def _make_paths(rng, batch, length, dim, width):
    dtype = np.float32 if width == 32 else np.float64
    steps = rng.standard_normal((batch, length, dim)) / np.sqrt(max(length, 1))
    return np.cumsum(steps, axis=1, dtype=np.float64).astype(dtype)


def _dp_instr(d, lx, ly):
    """Algorithmic FP64 instructions per fine cell."""
    f = 2.0 ** (lx + ly)
    return 3 + (d + 4) / f, 7 + (2 * d + 2) / f


def run_bench(task: str, *, batch=32, length=128, dim=4, dyadic_x=0, dyadic_y=0, reps=50,
              scalar_width=64, seed=0, peak_fma=None) -> BenchReport:
    """Run one task on cuda:0 and report the minimum device time over reps.

    kernel-*: `batch` aligned pairs (the reference's kernel_batch /
    kernel_batch_backward); gram-*: the symmetric Gram of `batch` paths
    (gram-value-grad: G and its gradient in one fused pass, cotangent ones).
    peak_fma (FMA/s) adds roofline_frac = algorithmic FMA / time / peak."""
    import torch

    from . import ops
    from .api import sig_kernel_gram_value_and_grad

    if task not in TASKS:
        raise InvalidArgument(f"unknown bench task {task!r}, expected one of {TASKS}")
    if reps < 1:
        raise InvalidArgument("reps must be >= 1")
    if batch < 1 or length < 2 or dim < 1:
        raise InvalidArgument("batch >= 1, length >= 2 and dim >= 1 required")
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", 0)
    shape = {"B": batch, "L": length, "d": dim, "dyadic_x": dyadic_x, "dyadic_y": dyadic_y}
    x = torch.as_tensor(_make_paths(rng, batch, length, dim, scalar_width), device=dev)
    m1, m2 = (length - 1) << dyadic_x, (length - 1) << dyadic_y
    i_fwd, i_bwd = _dp_instr(dim, dyadic_x, dyadic_y)
    if task.startswith("kernel"):
        y = torch.as_tensor(_make_paths(rng, batch, length, dim, scalar_width), device=dev)
        cells = batch * m1 * m2
        if task == "kernel-fwd":
            fn, work = (lambda: ops.forward_batch(x, y, dyadic_x, dyadic_y, 0, 1.0)), i_fwd
        else:
            fn = lambda: ops.backward_batch(x, y, dyadic_x, dyadic_y, 0, 1.0, None,  # noqa: E731
                                            want_values=True)
            work = i_fwd + i_bwd  # values and gradients, as kernel_batch_backward
    else:
        cells = batch * (batch + 1) // 2 * m1 * m2
        ones = torch.ones((batch, batch), dtype=torch.float64, device=dev)
        if task == "gram-fwd":
            fn, work = (lambda: ops.forward_gram(x, None, dyadic_x, dyadic_y, 0, 1.0)), i_fwd
        elif task == "gram-bwd":
            fn = lambda: ops.backward_gram(x, None, dyadic_x, dyadic_y, 0, 1.0, ones)  # noqa: E731
            work = i_bwd
        else:
            fn = lambda: sig_kernel_gram_value_and_grad(  # noqa: E731
                x, None, ones, (dyadic_x, dyadic_y))
            work = i_fwd + i_bwd
    fn()  # warm-up (workspaces; the kernels are precompiled)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    rep = BenchReport(task=task, shape=shape, repetitions=reps, times=times,
                      scalar_width=scalar_width, cells=int(cells))
    if peak_fma:
        rep.roofline_frac = cells * work / rep.minimum / peak_fma
    return rep
