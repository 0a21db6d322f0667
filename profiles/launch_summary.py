"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel total time and share (serialised, cold-cache: compare shares)."""
import collections
import csv
import sys


def summarise(path, top=15):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hdr], rows[hdr + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v for _, v in agg.values())
    out = []
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v / 1e6:10.3f} ms {100 * v / tot:5.1f}%  n={n:4d}  {k}")
    out.append(f"{tot / 1e6:10.3f} ms total")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15))
