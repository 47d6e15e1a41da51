"""Per-kernel SASS stall hotspots of one launch in an ncu report:
    python tools/ncu_kernel_hotspots.py report.ncu-rep LAUNCH_INDEX [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, launch, top=16):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(launch), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[0][1][:100])
    hdr = rows[1]
    ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot, byop, recs, st = 0, defaultdict(int), [], defaultdict(int)
    for r in rows[2:]:
        if len(r) <= max(sc):
            continue
        try:
            n = int(r[iall] or 0)
        except ValueError:
            continue
        tot += n
        toks = r[isrc].split()
        op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")).split(".")[0]
        byop[op] += n
        d = {hdr[i][6:]: int(r[i] or 0) for i in sc}
        for k, v in d.items():
            st[k] += v
        recs.append((n, r[ia][-5:], r[isrc][:64], d))
    print("samples", tot)
    print("stalls:", ", ".join(f"{k} {100 * v / max(1, sum(st.values())):.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    print("by op:", ", ".join(f"{k} {100 * v / max(1, tot):.1f}%" for k, v in sorted(byop.items(), key=lambda x: -x[1])[:12]))
    for n, a, s, d in sorted(recs, key=lambda x: -x[0])[:top]:
        t = sorted(d.items(), key=lambda x: -x[1])[:2]
        print(f"{n:8d} {a} {s:64s} {t}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 16)
