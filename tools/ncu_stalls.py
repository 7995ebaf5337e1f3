"""Stall-reason totals of an ncu --set full report over a SASS line range (all lines by default).

    python tools/ncu_stalls.py report.ncu-rep [first_line last_line]
"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw.split('"Kernel Name"')[1].split("\n", 1)[1])))
hdr, data = rows[0], rows[1:]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, len(data))
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {hdr[i]: sum(float(r[i] or 0) for r in data[lo:hi] if len(r) > i) for i in cols}
s = sum(tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"{k:24s} {v:8.0f} {100 * v / s:5.1f}%")
