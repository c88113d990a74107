"""Print registers/spills per kernel instance of one translation unit (dev tool)."""
import re
import subprocess
import sys

src = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-c", src, "-o", "/tmp/_regs.o", "-Xptxas", "-v"],
                   capture_output=True, text=True)
txt = r.stdout + r.stderr
for b in re.split(r"Compiling entry function '", txt)[1:]:
    name = b.split("'")[0]
    m = re.search(r"(fwd|bwd)_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)EL[ib](\d+)(?:ELi(\d+))?", name)
    if not m:
        continue
    regs = re.search(r"Used (\d+) registers", b).group(1)
    sp = re.search(r"(\d+) bytes spill stores", b).group(1)
    k, kind, DP, R, FR, F, a, bb = m.groups()
    line = f"{k} kind={kind} DP={DP} R={R} FR={FR} F={F} {'G/XW' if k == 'fwd' else 'CB'}={a} {bb or ''} regs={regs} spill={sp}"
    if filt in line:
        print(line)
