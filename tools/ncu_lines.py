"""Dev: per-source-line instruction / stall-sample totals of one kernel in an ncu report.
    python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
hdr = None
agg = collections.Counter()
samp = collections.Counter()
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        key = (cur, int(r[0]), r[1].strip()[:80])
        try:
            agg[key] += int(r[ie] or 0)
            samp[key] += int(r[ss] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
tots = sum(samp.values()) or 1
print(f"total instructions {tot}, stall samples {tots}")
for k, v in agg.most_common(top):
    print(f"{v / tot * 100:5.1f}% inst {samp[k] / tots * 100:5.1f}% samp  {k[0]}:{k[1]}  {k[2]}")
