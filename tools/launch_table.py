"""Per-kernel table from an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python tools/launch_table.py launches.csv [--ids]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
            out.append((int(d["ID"]), d["Kernel Name"], v))
    return out


def main():
    recs = load(sys.argv[1])
    if "--ids" in sys.argv:
        for i, k, v in recs:
            print(f"{i:5d} {v:10.1f} us  {k[:90]}")
        return
    agg = collections.OrderedDict()
    for _, k, v in recs:
        name = k.split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e3:9.3f} ms {n:5d} launches {100 * t / tot:5.1f}%  {k[:80]}")
    print(f"{tot / 1e3:9.3f} ms total")


if __name__ == "__main__":
    main()
