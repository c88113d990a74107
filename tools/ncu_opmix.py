"""Executed-instruction mix by SASS opcode from an ncu report's source page."""
import collections
import csv
import io
import subprocess
import sys

rep, kf = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kf}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie = h.index("Instructions Executed")
mix = collections.Counter()
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    op = r[1].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    op = op.split()[0].split(".")[0]
    mix[op] += int(r[ie])
tot = sum(mix.values())
print(f"total warp instructions {tot:.3e}")
for op, n in mix.most_common(25):
    print(f"  {op:10s} {n / tot * 100:5.1f}%")
