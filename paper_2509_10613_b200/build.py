"""Build the sm_100a shared library in-tree (paper_2509_10613_b200/_native/).

nvcc cross-compiles without a GPU.  Translation units compile in parallel;
the result is libsigkernel.so, loaded by ctypes (paper_2509_10613_b200/_lib.py).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_native")
SO = os.path.join(OUT, "libsigkernel.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-ccbin", "/usr/bin/g++", "--expt-relaxed-constexpr"]
SOURCES = ["sk_capi.cu", "sk_fwd_linear.cu", "sk_fwd_rbf.cu", "sk_fwd_delta.cu", "sk_fwd_f32.cu", "sk_fwd_short.cu",
           "sk_bwd_linear.cu", "sk_bwd_rbf.cu", "sk_bwd_wide.cu", "sk_bwd_xw_linear.cu", "sk_bwd_xw_rbf.cu", "sk_signature.cu", "sk_fwd_mma.cu", "sk_bwd_mma.cu",
           "sk_small.cu"]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "sigkernel.h")]


def _compile(src: str, extra: list[str], out: str = OUT) -> str:
    obj = os.path.join(out, os.path.splitext(src)[0] + ".o")
    newest = max(os.path.getmtime(p) for p in _deps())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False, extra: list[str] | None = None, out: str = OUT) -> str:
    """Compile every translation unit into `out` (default: the in-tree
    _native/; experiment variants with extra flags go to their own directory,
    selected at run time with SK_LIBSIGKERNEL)."""
    os.makedirs(out, exist_ok=True)
    so = os.path.join(out, "libsigkernel.so")
    extra = list(extra or [])
    if verbose:
        extra += ["-Xptxas", "-v"]
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra, out), SOURCES))
    if not os.path.exists(so) or os.path.getmtime(so) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", so, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return so


if __name__ == "__main__":
    # python -m paper_2509_10613_b200.build [-v] [--variant NAME -DFLAG ...]
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        name, flags = args[i + 1], [a for a in args[i + 2:] if a != "-v"]
        print(build(verbose="-v" in args, extra=flags, out=os.path.join(OUT, "variants", name)))
    else:
        print(build(verbose="-v" in args))
