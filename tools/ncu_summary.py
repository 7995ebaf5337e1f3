"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name."""
import collections
import csv
import sys


def summarise(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr, data = rows[hdr_i], rows[hdr_i + 1:]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    agg, tot = collections.defaultdict(lambda: [0, 0.0]), 0.0
    scale = {'nsecond': 1.0, 'ns': 1.0, 'usecond': 1e3, 'us': 1e3, 'msecond': 1e6, 'ms': 1e6, 'second': 1e9, 's': 1e9}
    for r in data:
        name = r[ki].split('(')[0].replace('<unnamed>::', '').replace('void ', '')[:56]
        v = float(r[vi].replace(',', '')) * scale[r[ui]]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    lines = [f"{'ms':>9} {'share':>6} {'n':>6} {'avg_us':>9}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        lines.append(f"{t / 1e6:9.3f} {100 * t / tot:5.1f}% {n:6d} {t / n / 1e3:9.1f}  {k}")
    lines.append(f"total {tot / 1e6:.3f} ms over {sum(n for n, _ in agg.values())} launches")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(summarise(p))
