"""Per-instruction stall hotspots from an ncu report's source page (SASS)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iall, inot = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Warp Stall Sampling (Not-issued Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
    tot = 0
    by_op = defaultdict(int)
    recs = []
    for r in rows[2:]:
        try:
            s = int(r[iall])
        except (ValueError, IndexError):
            continue
        tot += s
        op = r[isrc].split()[0] if r[isrc].split() else "?"
        if op.startswith("@"):
            op = r[isrc].split()[1]
        by_op[op.split(".")[0]] += s
        recs.append((s, int(r[inot] or 0), r[ia], r[isrc].strip()))
    print("total samples", tot)
    for op, s in sorted(by_op.items(), key=lambda x: -x[1])[:12]:
        print(f"{op:14s} {s:8d} {100.0 * s / max(tot, 1):5.1f}%")
    print("--- top instructions (all, not-issued)")
    for s, ni, a, src in sorted(recs, reverse=True)[:top]:
        print(f"{s:7d} {ni:7d} {a} {src}")
    extra = [h for h in hdr if "stall" in h.lower()][:60]
    print(extra)


if __name__ == "__main__":
    main(sys.argv[1])
