"""Summarise an ncu report: key metrics + top stall reasons + hottest SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""


def run(args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
hdr = raw[0]
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__inst_executed_op_shfl.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second"]
for row in raw[2:]:
    name = row[hdr.index("Kernel Name")]
    if kfilter not in name:
        continue
    print("==", name[:110])
    for w in want:
        if w in hdr:
            print(f"  {w} = {row[hdr.index(w)]} {raw[1][hdr.index(w)]}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(row[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("  stalls (cycles per issued instr):", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:7]))

src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv"] + (["-k", f"regex:{kfilter}"] if kfilter else [])))))
if len(src) > 2:
    h = src[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in src[2:] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in data) or 1
    print("  hottest SASS (share of stall samples):")
    for r in sorted(data, key=lambda r: -int(r[si]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
        print(f"   {int(r[si]) / tot * 100:5.1f}%  {r[1].strip()[:90]}")
