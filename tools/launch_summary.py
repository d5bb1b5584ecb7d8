"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total device time and share."""
import collections
import csv
import sys


def summarize(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[0] == "ID":
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {sum(v[0] for v in agg.values())}, total device time {tot / 1e6:.3f} ms (cold-cache, serialised)"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:24s} {v[0]:6d} launches {v[1] / 1e6:9.3f} ms {100 * v[1] / tot:6.1f}%  avg {v[1] / v[0] / 1e3:8.1f} us")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
