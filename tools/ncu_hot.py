"""Top SASS instructions by warp-stall samples from an ncu report (``--page source``)."""
import csv
import io
import subprocess
import sys


def hot(path, top=40, kernel_idx=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = raw.split('"Kernel Name"')[1:]
    rows = list(csv.reader(io.StringIO(blocks[kernel_idx].split("\n", 1)[1])))
    hdr, data = rows[0], rows[1:]
    si, ni = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    tot = sum(float(r[si] or 0) for r in data if len(r) > si)
    out = []
    for i, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0) if len(x[1]) > si else 0)[:top]:
        out.append(f"{100 * float(r[si]) / tot:5.1f}%  #{i:5d} {r[ni].strip()[:90]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(hot(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40))
