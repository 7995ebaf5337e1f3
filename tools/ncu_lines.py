"""Per-CUDA-source-line warp-stall samples of an ncu --set full report (top N lines), from the
source page in "cuda,sass" mode (rows whose first column is a source line number).

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
out, fname = [], "?"
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0].isdigit() and len(r) > 4 and r[2] == "-" and r[4] not in ("", "0"):
        out.append((float(r[4]), fname, r[0], r[1][:100]))
tot = sum(x[0] for x in out) or 1
for v, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{ln:5s} {src}")
