"""Group an ncu source page (SASS) into runs of equal execution count: where the instructions go.
    python tools/ncu_blocks.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia] or 0) for r in data)
print("total warp instructions", tot)
blocks = []
for i, r in enumerate(data):
    c = int(r[ia] or 0)
    if blocks and blocks[-1][1] == c:
        blocks[-1][2] += 1
        blocks[-1][3] += int(r[iss] or 0)
    else:
        blocks.append([i, c, 1, int(r[iss] or 0), r[isrc].strip()[:60]])
blocks.sort(key=lambda b: -b[1] * b[2])
for b in blocks[:top]:
    print(f"line {b[0]:5d} count {b[1]:10d} x {b[2]:4d} instr = {b[1] * b[2] / tot * 100:5.1f}%  stall-samples {b[3]:6d}  | {b[4]}")
