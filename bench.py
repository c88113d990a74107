"""Benchmark: signature-kernel Gram forward+backward (fp64) on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  N>1 runs under torchrun, one rank per GPU (NCCL).

Workload (default --config c3, BASELINE.json configs[2]): symmetric
sig_kernel_gram of 1024 Brownian paths, L=512, d=16, dyadic order 0, linear
static kernel, fp64 forward + exact backward with cotangent ones (the
reference default, kernel_grad.py:81-82).  A "step" = the Gram G AND the
gradient dF/dX of F = sum G, computed by ONE fused value + gradient pass
(sig_kernel_gram_value_and_grad; the Gram counterpart of the reference's
kernel_batch_backward, which returns values with the gradients,
kernel_grad.py:64-98).  The autograd split (forward kernel, then backward
kernel) is reported beside it ("unfused", "e2e_autograd").  With N GPUs the
same Gram is sharded by balanced row blocks (strong scaling) and assembled
with NCCL all-gathers.

  value  = solved PDE cells per second (device-resident inputs, device timed,
           max over ranks); Gram entries/s reported beside it
  e2e    = the same step through the public API (sig_kernel_gram_value_and_grad)
           from pinned host memory: H2D of X and D2H of G and dF/dX inside
           the timed region
  roofline: the fused kernel vs the FP64 pipe (DMMA + DFMA), algorithmic DP
           instructions per cell (I_fwd + I_bwd), peak measured
           live with a DFMA probe on this GPU
  cpu_baseline: the C oracle (restatement of the reference algorithm,
           OpenMP over pairs, all host threads) on a bounded sub-Gram

`--impl reference` times the reference's CPU algorithm on the same metric with
all host threads: the C oracle port (the line's value; faster than stock
sigcore, so the ratio is conservative) and, beside it, the unmodified sigcore
(Python + numba, pip-installed into baseline/_ref) on the same sub-Gram step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("sig-kernel PDE cells/sec and Gram entries/sec (fwd+bwd, fp64) vs roofline & CPU")

CONFIGS = {
    # name: (n, L, d, lam, description)
    "c3": (1024, 512, 16, 0,
           "sig_kernel_gram 1024x1024, length=512, dim=16, fp64 forward+backward on 1xB200 "
           "(BASELINE configs[2])"),
    "c5": (8192, 1024, 8, 0,
           "sig_kernel_gram 8192x8192, length=1024, dim=8, forward+backward sharded "
           "(BASELINE configs[4])"),
}


def make_paths(rng, batch, length, dim):
    """Reference bench generator (sigcore/bench.py:53-56), fp64."""
    steps = rng.standard_normal((batch, length, dim)) / np.sqrt(max(length, 1))
    return np.cumsum(steps, axis=1, dtype=np.float64)


def dp_instr_per_cell(d, lam1, lam2):
    """Algorithmic FP64 instructions per fine cell:
    I_fwd = 3 + (d+4)/2^(l1+l2),  I_bwd = 7 + (2d+2)/2^(l1+l2)."""
    s = 2.0 ** (lam1 + lam2)
    return 3 + (d + 4) / s, 7 + (2 * d + 2) / s


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(n_sample, L, d, lam, budget_s=10.0):
    """Oracle (C restatement of the reference, OpenMP) fwd+bwd on a sub-Gram."""
    from oracle import oracle as orc
    orc.build()
    rng = np.random.default_rng(0)
    X = make_paths(rng, n_sample, L, d)
    C = np.ones((n_sample, n_sample))
    threads = os.cpu_count() or 1
    orc.gram_backward(X[:2], None, C[:2, :2], lam, lam, threads=threads)  # warm
    pairs = n_sample * (n_sample + 1) // 2
    cells = pairs * ((L - 1) << lam) ** 2
    reps, t0 = 0, time.perf_counter()
    while True:
        orc.gram_backward(X, None, C, lam, lam, threads=threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= 50:
            break
    return {"value": cells * reps / el, "unit": "cells/s", "cores": threads, "kind": "port",
            "sample": f"symmetric sub-Gram {n_sample}x{n_sample} (L={L}, d={d}, lambda={lam}) "
                      f"fwd+bwd, {reps} rep(s) in {el:.1f}s; oracle/sk_oracle.c (restates "
                      f"sigcore goursat_grid+goursat_backward per pair)",
            "entries_per_s": n_sample * n_sample * reps / el}


def small_call_latency(dev, n=2000):
    """Per-call cost of the small-problem path (BASELINE configs[0]: 32 pairs,
    L=64, d=4, lambda 0) through the public API sig_kernel: host time per call
    (calls enqueued back to back, one sync) and one blocking call (enqueue,
    kernel, sync).  Not part of the timed step."""
    import torch
    import paper_2509_10613_b200 as sk
    rng = np.random.default_rng(0)
    x = torch.as_tensor(make_paths(rng, 32, 64, 4), device=dev)
    y = torch.as_tensor(make_paths(rng, 32, 64, 4), device=dev)
    for _ in range(100):
        sk.sig_kernel(x, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        sk.sig_kernel(x, y)
    torch.cuda.synchronize()
    per_call = (time.perf_counter() - t0) / n
    ts = []
    for _ in range(200):
        t1 = time.perf_counter()
        sk.sig_kernel(x, y)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t1)
    return {"config": "BASELINE configs[0]: sig_kernel fwd, 32 pairs, L=64, d=4, lambda=0",
            "us_per_call_pipelined": per_call * 1e6,
            "us_blocking_median": statistics.median(ts) * 1e6,
            "api": "paper_2509_10613_b200.sig_kernel"}


def config_dict(name, world):
    """The workload's config (identical on both arms of the bench)."""
    n, L, d, lam, desc = CONFIGS[name]
    return {"workload": desc, "n": n, "L": L, "d": d, "dyadic_order": lam,
            "static_kernel": "linear", "cotangent": "ones", "symmetric": True,
            "parallelism": f"gram row blocks x{world}",
            "l2": "flushed between timed steps (256 MiB write)"}


def run_reference(args, rank, world):
    """--impl reference: the reference CPU algorithm (oracle port), rank 0 only."""
    if rank != 0:
        return
    n, L, d, lam, desc = CONFIGS[args.config]
    n_sample = 24 if args.config == "c3" else 8
    from oracle import oracle as orc
    orc.build()
    rng = np.random.default_rng(0)
    X = make_paths(rng, n_sample, L, d)
    C = np.ones((n_sample, n_sample))
    threads = os.cpu_count() or 1
    pairs = n_sample * (n_sample + 1) // 2
    cells = pairs * ((L - 1) << lam) ** 2
    for _ in range(args.warmup):
        orc.gram_backward(X[:4], None, C[:4, :4], lam, lam, threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.gram_backward(X, None, C, lam, lam, threads=threads)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = cells / t
    sample = (f"symmetric sub-Gram {n_sample}x{n_sample} of the {desc} workload per step "
              f"(cells/s is size-independent per pair; full config extrapolates linearly)")
    stock = stock_reference(X[:8], C[:8, :8], lam, threads)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "cells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference _make_paths, seed 0)",
        "config": config_dict(args.config, world),
        "sample": f"{n_sample}x{n_sample} symmetric sub-Gram per step",
        "gram_entries_per_s": n_sample * n_sample / t,
        "cpu_baseline": {"value": value, "unit": "cells/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "value_source": "the C port (faster than stock sigcore, so the GPU/CPU ratio is "
                        "conservative); stock sigcore timed beside it in stock_reference",
        "stock_reference": stock,
    }), flush=True)


def stock_reference(X, C, lam, threads):
    """The unmodified reference (sigcore, Python + numba, installed into
    baseline/_ref) on the same sub-Gram step: kernel_gram (kernel.py:151-180)
    for G, then kernel_batch_backward (kernel_grad.py:64-98) over the upper
    triangle's pairs for dF/dX (sigcore has no Gram backward).  Reported beside
    the port; None when baseline/_ref or numba is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "sigcore")):
        return {"unavailable": "baseline/_ref/sigcore not installed"}
    sys.path.insert(0, ref)
    try:
        from sigcore.kernel import KernelConfig, kernel_gram
        from sigcore.kernel_grad import kernel_batch_backward
    except Exception as e:  # noqa: BLE001 - report, do not fail the arm
        return {"unavailable": f"import sigcore failed: {type(e).__name__}: {e}"}
    finally:
        sys.path.remove(ref)
    n, L = X.shape[0], X.shape[1]
    cfg = KernelConfig(lam, lam)
    ia, ib = np.triu_indices(n)

    def step():
        kernel_gram(X, None, cfg, threads=threads)
        kernel_batch_backward(X[ia], X[ib], cfg, C[ia, ib], threads=threads)

    kernel_gram(X[:2], None, cfg, threads=threads)  # numba JIT compile, untimed
    kernel_batch_backward(X[:1], X[:1], cfg, None, threads=threads)
    t0 = time.perf_counter()
    step()
    t = time.perf_counter() - t0
    cells = len(ia) * ((L - 1) << lam) ** 2
    return {"value": cells / t, "unit": "cells/s", "cores": threads, "kind": "reference",
            "ms_per_step": t * 1e3,
            "sample": f"symmetric sub-Gram {n}x{n}: sigcore.kernel_gram + "
                      f"kernel_batch_backward over its {len(ia)} upper-triangle pairs"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    # test hook: SK_BENCH_ONE_GPU=1 puts every rank on cuda:0 and uses gloo, so
    # the N > 1 code path (row blocks, all-gathers, max over ranks) can be
    # exercised on a one-GPU box (its timings are meaningless)
    one_gpu = os.environ.get("SK_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_2509_10613_b200 as sk
    from paper_2509_10613_b200 import gram_dist, ops

    n, L, d, lam, desc = CONFIGS[args.config]
    rng = np.random.default_rng(0)
    Xh = make_paths(rng, n, L, d)
    X = torch.as_tensor(Xh, device=dev)
    C = torch.ones((n, n), dtype=torch.float64, device=dev)
    ranges = gram_dist.row_blocks(n, world, rank, True)
    my_pairs = gram_dist.pair_count(ranges, n, True)
    total_pairs = n * (n + 1) // 2
    cells_pair = ((L - 1) << lam) ** 2
    i_fwd, i_bwd = dp_instr_per_cell(d, lam, lam)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def step_device(ev=None):
        """Device-resident step: ONE fused value + gradient pass (G and dF/dX of
        F = sum C * G, C = ones) -- the Gram counterpart of the reference's
        kernel_batch_backward, which returns values with the gradients.
        Optionally records (start, end) events."""
        if ev is not None:
            ev[0].record()
        if world == 1:
            parts = [ops.value_and_grad_gram(X, None, lam, lam, 0, 1.0, C)[0]]
            gx = None
        else:  # exact accumulators: bitwise the one-GPU gradient (gram_dist)
            acc = ops.GradAcc(n, L, d, dev).init(C, n, n, True)
            parts = [ops.value_and_grad_gram(X, None, lam, lam, 0, 1.0, C, rows=rg,
                                             acc_x=acc)[0] for rg in ranges]
        if ev is not None:
            ev[1].record()
        if world > 1:
            local_rows = torch.cat(parts, 0)
            ranges_all = [gram_dist.row_blocks(n, world, r, True) for r in range(world)]
            G = gram_dist._gather_rows(local_rows, ranges_all, n, n, group, symmetric=True)
            ops.mirror_upper(G)
            gx = gram_dist._allreduce_acc(acc, group).finalize()
        return parts, gx

    def step_unfused(ev):
        """The autograd-style step: forward Gram, then the backward (which
        re-solves the forward for its checkpoints).  Reported beside the fused
        step; ev = (start, fwd_end, end)."""
        ev[0].record()
        parts = [ops.forward_gram(X, None, lam, lam, 0, 1.0, rows=rg) for rg in ranges]
        ev[1].record()
        gx = torch.zeros_like(X)
        for rg in ranges:
            ops.backward_gram(X, None, lam, lam, 0, 1.0, C, rows=rg, grad_x=gx)
        ev[2].record()
        return parts, gx

    # warmup (also sizes workspaces / JIT-free: kernels are precompiled)
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    peak_fma = ops.dfma_peak()  # live FP64 roofline denominator on this GPU

    sampler = ClockSampler(local)
    sampler.start()
    step_ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (256 MiB > 126 MB L2)
        barrier()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e_end = torch.cuda.Event(enable_timing=True)
        step_device(ev)
        e_end.record()
        torch.cuda.synchronize()
        barrier()
        step_ms.append(ev[0].elapsed_time(e_end))
        kern_ms = ev[0].elapsed_time(ev[1])
    clocks = sampler.stop()
    # unfused split (forward kernel, then backward kernel), fewer steps
    fwd_ms, bwd_ms = [], []
    for _ in range(max(1, min(args.steps, 2))):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        step_unfused(ev)
        torch.cuda.synchronize()
        barrier()
        fwd_ms.append(ev[0].elapsed_time(ev[1]))
        bwd_ms.append(ev[1].elapsed_time(ev[2]))

    t_step = sum(step_ms) / len(step_ms) / 1e3
    t_bwd = sum(bwd_ms) / len(bwd_ms) / 1e3
    t_fwd = sum(fwd_ms) / len(fwd_ms) / 1e3
    if world > 1:
        tt = torch.tensor([t_step, t_bwd, t_fwd], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_bwd, t_fwd = tt.tolist()

    total_cells = total_pairs * cells_pair
    value = total_cells / t_step
    my_cells = my_pairs * cells_pair
    # the fused kernel does the forward (values) and the backward: algorithmic
    # work = (I_fwd + I_bwd) DP instructions per cell
    achieved = my_cells * (i_fwd + i_bwd) * 2 / t_step / 1e12  # FMA-equivalent TFLOP/s
    peak = 2 * peak_fma / 1e12

    # ---- e2e through the public API, host buffers, copies inside the region
    e2e = None
    e2e_autograd = None
    if not args.no_e2e:
        Xpin = torch.from_numpy(Xh).pin_memory()
        Gh = torch.empty((n, n), dtype=torch.float64).pin_memory()
        gh = torch.empty_like(Xpin).pin_memory()

        def step_e2e():  # the fused public call (cotangent ones = its default)
            Xd = Xpin.to(dev, non_blocking=True)
            if world > 1:
                G, g, _ = gram_dist.value_and_grad_sharded(Xd, dyadic_order=lam, group=group)
            else:
                G, g, _ = sk.sig_kernel_gram_value_and_grad(Xd, dyadic_order=lam)
            Gh.copy_(G, non_blocking=True)
            gh.copy_(g, non_blocking=True)

        def step_autograd():  # sig_kernel_gram + torch autograd (forward, then backward)
            Xd = Xpin.to(dev, non_blocking=True).requires_grad_(True)
            if world > 1:
                G = gram_dist.sig_kernel_gram_sharded(Xd, dyadic_order=lam)
            else:
                G = sk.sig_kernel_gram(Xd, dyadic_order=lam)
            G.sum().backward()  # cotangent ones
            Gh.copy_(G.detach(), non_blocking=True)
            gh.copy_(Xd.grad, non_blocking=True)

        def timed(fn, reps):
            fn()
            torch.cuda.synchronize()
            ms = []
            for _ in range(reps):
                flush.fill_(1.0)
                barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                barrier()
                ms.append(a.elapsed_time(b))
            t = sum(ms) / len(ms) / 1e3
            if world > 1:
                tt = torch.tensor([t], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = tt.item()
            return t

        t_e2e = timed(step_e2e, max(1, min(args.steps, 3)))
        t_ag = timed(step_autograd, 1)
        io = {"h2d_bytes_per_step": int(Xh.nbytes),
              "d2h_bytes_per_step": int(Gh.numel() * 8 + gh.numel() * 8)}
        e2e = {"value": total_cells / t_e2e, "unit": "cells/s", **io,
               "ms_per_step": t_e2e * 1e3,
               "api": "paper_2509_10613_b200.sig_kernel_gram_value_and_grad (fused G + dF/dX)"
                      + (" via gram_dist.value_and_grad_sharded" if world > 1 else "")}
        e2e_autograd = {"value": total_cells / t_ag, "unit": "cells/s", **io,
                        "ms_per_step": t_ag * 1e3,
                        "api": "paper_2509_10613_b200.sig_kernel_gram + torch autograd"
                               + (" (gram_dist sharded)" if world > 1 else "")}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except (OSError, ValueError):
            traffic = None

    latency = small_call_latency(dev) if (rank == 0 and world == 1 and not args.no_e2e) else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(24 if args.config == "c3" else 8, L, d, lam)

    if rank == 0:
        # our kernels per step (ncu launch list, profiles/r02_launches_c3_final.csv):
        # one GPU: prep_sides, fix_init (exact accumulators), gram_bwd_mma,
        # fix_finalize, mirror_upper; sharded: accumulator init, per row range
        # prep + fused kernel + block mirror, then the mirror after the gather
        # and the finalize
        launches_per_step = 5 if world == 1 else 3 * len(ranges) + 3
        out = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic Brownian paths (reference _make_paths generator, seed 0)",
            "config": config_dict(args.config, world),
            "gram_entries_per_s": n * n / t_step,
            "step": "one fused value + gradient pass per row block (G and dF/dX; the Gram "
                    "counterpart of the reference's kernel_batch_backward, which returns values "
                    "with gradients, kernel_grad.py:64-98)",
            "kernel_ms": kern_ms,
            "unfused": {"fwd_ms": t_fwd * 1e3, "bwd_ms": t_bwd * 1e3,
                        "ms_per_step": (t_fwd + t_bwd) * 1e3,
                        "value": total_cells / (t_fwd + t_bwd),
                        "what": "forward Gram kernel, then the backward kernel (the torch "
                                "autograd split; the backward re-solves the forward)"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "kernel": "gram_bwd_mma in value+gradient mode (FP64 tensor-core DMMA "
                                   "for <dx,dy>, gx, gy + DFMA wavefronts: forward with "
                                   "checkpoints, block recompute, reverse sweep)",
                         "pipe": "FP64: DMMA (mma.m8n8k4.f64) and DFMA share one pipe on B200 "
                                 "(tools/dmma_probe.cu), so the FP64 peak bounds both",
                         "work": f"{i_fwd:g} + {i_bwd:g} DP instr/cell (SURVEY 8d I_fwd + I_bwd) "
                                 f"x {my_cells} cells per launch; FMA-equivalent flops = 2 x DP "
                                 f"instr; timed over the step (the kernel is "
                                 f"{100 * kern_ms / (t_step * 1e3):.1f} % of it)",
                         "peak_source": "live DFMA probe on this GPU (MEASURED_PEAKS.json "
                                        "has no FP64 figure)",
                         # what the kernel actually issues per cell (lambda = 0): forward
                         # with checkpoints (7 DFMA + d DMMA-FMA), block recompute (7 + d),
                         # adjoint sweep (13), gx/gy maps (2d on DMMA)
                         "executed_fma_per_cell": 27 + 4 * d,
                         "executed_frac": my_cells * (27 + 4 * d) / t_step / peak_fma},
            "e2e_autograd": e2e_autograd,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "latency_c1": latency,
            "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
