"""GPU-backed command line for the signature-kernel path.

    python -m paper_2509_10613_b200.cli kernel --input x.sgt --input2 y.sgt \
        [--dyadic-x N] [--dyadic-y N] [--output k.sgt] \
        [--cotangent c.sgt --grad-output-x gx.sgt --grad-output-y gy.sgt]
    python -m paper_2509_10613_b200.cli gram --input x.sgt [--input2 y.sgt] --output g.sgt
    python -m paper_2509_10613_b200.cli bench --task gram-value-grad --batch 64 --length 256 \
        --dim 8 [--reps N] [--roofline] [--json] [--output r.json]

Same subcommands, flags, file format and exit codes (0 ok, 2 usage, 1 data
error) as the reference CLI's `kernel` and `gram` (sigcore/cli.py:53-73,
137-164, 198-207), so the reference's CLI tests and its TypeScript bindings
(which drive the CLI through SGT1 files) run against the B200 kernels.
Extension: --rbf-sigma S selects the RBF static kernel.  --threads is
accepted for compatibility and ignored.
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import sigcore_compat as sc
from .errors import FormatError, InvalidArgument, InvalidState, NativeUnavailable
from .sgt_io import read_array, write_array


def _common(p):
    p.add_argument("--threads", type=int, default=None, help="accepted, ignored (GPU)")
    p.add_argument("--dtype", choices=("f32", "f64"), default=None,
                   help="force the storage width of the inputs")
    p.add_argument("--rbf-sigma", type=float, default=None,
                   help="use the RBF static kernel with this sigma (default: linear)")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="sigkernel-b200",
                                 description="Signature kernels on B200 (sm_100a)")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("kernel", help="pairwise signature kernels of two batches")
    p.add_argument("--input", required=True)
    p.add_argument("--input2", required=True)
    p.add_argument("--dyadic-x", type=int, default=0)
    p.add_argument("--dyadic-y", type=int, default=0)
    p.add_argument("--output", default=None, help="write values to a file instead of stdout")
    p.add_argument("--cotangent", default=None, help="dF/dk per pair; triggers the backward")
    p.add_argument("--grad-output-x", default=None)
    p.add_argument("--grad-output-y", default=None)
    _common(p)
    p = sub.add_parser("gram", help="Gram matrix of kernel values")
    p.add_argument("--input", required=True)
    p.add_argument("--input2", default=None, help="second batch (default: symmetric)")
    p.add_argument("--dyadic-x", type=int, default=0)
    p.add_argument("--dyadic-y", type=int, default=0)
    p.add_argument("--output", required=True)
    _common(p)
    # the reference's `bench` (sigcore/cli.py:81-92, bench.py:59-98) on the GPU
    # kernels, with Gram tasks; report: schemas/bench_report_gpu.schema.json
    from .bench_tasks import TASKS
    p = sub.add_parser("bench", help="time a task on the GPU; minimum over repetitions")
    p.add_argument("--task", choices=TASKS, required=True)
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--length", type=int, default=128)
    p.add_argument("--dim", type=int, default=4)
    p.add_argument("--dyadic-x", type=int, default=0)
    p.add_argument("--dyadic-y", type=int, default=0)
    p.add_argument("--reps", type=int, default=50)
    p.add_argument("--roofline", action="store_true",
                   help="measure the FP64 peak live and report roofline_frac")
    p.add_argument("--json", action="store_true", help="print the report as JSON")
    p.add_argument("--output", default=None, help="also write the JSON report here")
    _common(p)
    return ap


def _load(path, dtype_flag):
    a = read_array(path)
    if dtype_flag is not None:
        a = a.astype(np.float32 if dtype_flag == "f32" else np.float64)
    return a


def _static(args):
    if args.rbf_sigma is None:
        return None
    from .api import RBFKernel
    return RBFKernel(args.rbf_sigma)


def _kernel(args) -> int:
    x = _load(args.input, args.dtype)
    y = _load(args.input2, args.dtype)
    cfg = sc.KernelConfig(args.dyadic_x, args.dyadic_y)
    static = _static(args)
    if args.cotangent is not None:
        cot = read_array(args.cotangent)
        if static is None:
            values, gx, gy = sc.kernel_batch_backward(x, y, cfg, cot)
        else:
            values, gx, gy = _rbf_backward(x, y, cfg, cot, static)
        write_array(gx, args.grad_output_x)
        write_array(gy, args.grad_output_y)
    else:
        squeeze = np.asarray(x).ndim == 2
        if static is None:
            values = sc.kernel_batch(x, y, cfg)
        else:
            values = _rbf_forward(x, y, cfg, static)
        if squeeze:
            values = values[0]
    if args.output is not None:
        write_array(np.atleast_1d(values), args.output)
    else:
        for v in np.atleast_1d(values):
            print(repr(float(v)))
    return 0


def _torch_paths(a):
    import torch
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2:
        a = a[None]
    return torch.as_tensor(a, device="cuda")


def _rbf_forward(x, y, cfg, static):
    from . import ops
    kind, sigma = ops.static_kind(static)
    return ops.forward_batch(_torch_paths(x), _torch_paths(y), cfg.dyadic_x, cfg.dyadic_y,
                             kind, sigma).cpu().numpy()


def _rbf_backward(x, y, cfg, cot, static):
    import torch
    from . import ops
    kind, sigma = ops.static_kind(static)
    squeeze = np.asarray(x).ndim == 2
    c = torch.as_tensor(np.atleast_1d(np.asarray(cot, dtype=np.float64)), device="cuda")
    v, gx, gy = ops.backward_batch(_torch_paths(x), _torch_paths(y), cfg.dyadic_x, cfg.dyadic_y,
                                   kind, sigma, c, want_values=True)
    v, gx, gy = v.cpu().numpy(), gx.cpu().numpy(), gy.cpu().numpy()
    return (v[0], gx[0], gy[0]) if squeeze else (v, gx, gy)


def _gram(args) -> int:
    x = _load(args.input, args.dtype)
    y = None if args.input2 is None else _load(args.input2, args.dtype)
    cfg = sc.KernelConfig(args.dyadic_x, args.dyadic_y)
    static = _static(args)
    if static is None:
        G = sc.kernel_gram(x, y, cfg)
    else:
        from . import ops
        kind, sigma = ops.static_kind(static)
        G = ops.forward_gram(_torch_paths(x), None if y is None else _torch_paths(y),
                             cfg.dyadic_x, cfg.dyadic_y, kind, sigma).cpu().numpy()
    write_array(G, args.output)
    return 0


def _bench(args) -> int:
    from . import ops
    from .bench_tasks import run_bench
    peak = ops.dfma_peak() if args.roofline else None
    report = run_bench(args.task, batch=args.batch, length=args.length, dim=args.dim,
                       dyadic_x=args.dyadic_x, dyadic_y=args.dyadic_y, reps=args.reps,
                       scalar_width=32 if args.dtype == "f32" else 64, peak_fma=peak)
    text = report.to_json(indent=2)
    if args.output is not None:
        with open(args.output, "w") as fh:
            fh.write(text + "\n")
    if args.json:
        print(text)
    else:
        print(f"{report.task} shape={report.shape} reps={report.repetitions} "
              f"min={report.minimum:.6f}s cells/s={report.cells_per_s:.3e}")
    return 0


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    if args.command == "kernel" and args.cotangent is not None:
        if args.grad_output_x is None or args.grad_output_y is None:
            parser.error("--cotangent requires --grad-output-x and --grad-output-y")
    try:
        return {"kernel": _kernel, "gram": _gram, "bench": _bench}[args.command](args)
    except (InvalidArgument, InvalidState, FormatError, NativeUnavailable, OSError) as exc:
        print(f"sigkernel-b200: error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
