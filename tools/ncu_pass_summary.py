"""Per-kernel summary of the LAST profiled pass of an ncu launch list (tools/profile_iter.py under
`ncu --metrics gpu__time_duration.sum --csv`): launches from the last encoder call (k_enc_embed)
on, torch's own elementwise kernels excluded.

    python tools/ncu_pass_summary.py LABEL=launches.csv [LABEL=launches.csv ...]
"""
import collections
import csv
import sys

SCALE = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}


def summarise(label: str, path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    recs = [(r[ki].split('(')[0].replace('<unnamed>::', '').replace('void ', ''),
             float(r[vi].replace(',', '')) * SCALE[r[ui]]) for r in data]
    start = max(i for i, (n, _) in enumerate(recs) if n.startswith('k_enc_embed'))
    recs = [(n, t) for n, t in recs[start:] if not n.startswith(('at::', 'elementwise_kernel', 'vectorized'))]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, t in recs:
        agg[n][0] += 1
        agg[n][1] += t
    tot = sum(t for _, t in recs)
    out = [f"== {label}: {len(recs)} launches, {tot / 1e3:.3f} ms serialised",
           f"{'us':>10}  share    n  kernel"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{t:10.1f} {100 * t / tot:5.1f}% {c:4d}  {n}")
    return "\n".join(out)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        label, path = arg.split('=', 1)
        print(summarise(label, path))
        print()
