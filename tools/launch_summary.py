"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per
kernel launches, total time and share (cold-cache, serialised by ncu: compare
shares, not absolutes)."""
import collections
import csv
import io
import re
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def short(name):
    name = re.sub(r"^void ", "", name)
    base = name.split("(")[0]
    return base[:100]


def main(path, out=None):
    text = open(path).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(l for l in text[start:] if l.startswith('"'))))
            if r.get("Metric Name") == "gpu__time_duration.sum" and r.get("ID") != "ID"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        ms = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = [f"launch list: {path}  ({len(rows)} launches, {tot:.1f} ms total under ncu)"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[1]:10.2f} ms {100 * v[1] / tot:5.1f}%  {v[0]:6d} launches  {k}")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
