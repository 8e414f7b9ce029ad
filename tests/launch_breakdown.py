"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per epoch."""
import collections
import csv
import re
import sys


def main(path, n_timed=2, tail_epochs=4):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    names = [r[ki] for r in data]
    vals = [float(r[vi].replace(",", "")) for r in data]
    idx = [i for i, n in enumerate(names) if "plan_frozen" in n]
    # the timed epochs are followed by the e2e run: 2 warm-up + --steps (2) epochs
    s, e = idx[-(n_timed + tail_epochs)], idx[-tail_epochs]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in zip(names[s:e], vals[s:e]):
        m = re.search(r"(k_\w+|at::\w+|ncclDevKernel\w*)(<[^>]*>)?", n)
        k = (m.group(1) + (m.group(2) or "")) if m else n[:50]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v for _, v in agg.values())
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} {c // n_timed:4d}/epoch {v / n_timed / 1e3:9.1f} us/epoch {100 * v / tot:5.1f}%")
    print(f"{'total':44s} {'':9s} {tot / n_timed / 1e3:9.1f} us/epoch")


if __name__ == "__main__":
    main(sys.argv[1])
