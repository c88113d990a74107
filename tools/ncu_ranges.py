"""Stall samples / instructions of an ncu report summed over source-line ranges
of one file: python tools/ncu_ranges.py rep.ncu-rep file.cuh a-b c-d ..."""
import csv
import io
import subprocess
import sys

rep, fname, spans = sys.argv[1], sys.argv[2], sys.argv[3:]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, rows = None, None, []
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        cur = rec[1].rsplit("/", 1)[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or len(rec) < 8 or rec[2] != "-":
        continue
    try:
        s = int(rec[hdr.index("Warp Stall Sampling (All Samples)")])
        i = int(rec[hdr.index("Instructions Executed")])
    except ValueError:
        continue
    rows.append((cur, int(rec[0]), s, i))
ts = sum(r[2] for r in rows) or 1
ti = sum(r[3] for r in rows) or 1
for sp in spans:
    a, b = map(int, sp.split("-"))
    s = sum(r[2] for r in rows if r[0] == fname and a <= r[1] <= b)
    i = sum(r[3] for r in rows if r[0] == fname and a <= r[1] <= b)
    print(f"{fname}:{sp:12s} samples {100 * s / ts:5.1f}%  instructions {100 * i / ti:5.1f}%")
other = sum(r[2] for r in rows if r[0] != fname)
print(f"other files: samples {100 * other / ts:5.1f}%")
