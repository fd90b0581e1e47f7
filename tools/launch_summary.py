"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import io
import sys

UNIT = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}


def main(path, frames=1.0):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.OrderedDict()
    for r in rows:
        name = r["Kernel Name"].split("(")[0]
        name = name.replace("gsr::", "").split("::")[-1][:60]
        v = float(r["Metric Value"].replace(",", "")) * UNIT[r["Metric Unit"]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"{len(rows)} launches, {tot / 1e3 / frames:.1f} us per frame (ncu, serialised, cold)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e3 / frames:9.1f} us/frame {c / frames:6.1f} launches/frame "
              f"{100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
