"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel totals and shares of the device time."""
import collections
import csv
import json
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        k = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", "")) * UNIT.get(r[iu], 1e-6)
        tot[k] = tot.get(k, 0.0) + v
        cnt[k] += 1
    s = sum(tot.values())
    out = [{"kernel": k, "launches": cnt[k], "ms": round(v, 3), "share": round(v / s, 4)}
           for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    print(json.dumps({"total_ms": round(s, 3), "launches": sum(cnt.values()), "kernels": out}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
