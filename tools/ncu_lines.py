"""Per-source-line instructions and stall samples from an ncu report (cuda,sass view)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("Function Name",) or len(rec) < 8 or rec[2] != "-":
        continue
    try:
        samp = int(rec[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(rec[hdr.index("Instructions Executed")])
    except ValueError:
        continue
    rows.append((samp, inst, f"{fname}:{rec[0]}", rec[1].strip()[:80]))
ts = sum(r[0] for r in rows) or 1
ti = sum(r[1] for r in rows) or 1
print(f"total samples {ts}, warp instructions {ti:.3e}")
for s, i, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst  {loc:22s} {src}")
