"""Per-source-line warp-stall samples of one launch in an ncu report (needs
-lineinfo / --import-source): the top lines with their dominant stall reasons.
    python tools/ncu_lines.py report.ncu-rep LAUNCH_INDEX [top]"""
import csv
import io
import subprocess
import sys


def main(path, launch, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", str(launch), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, lines, total = None, None, [], 0
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or r[0] in ("", "Function Name"):
            continue
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        stalls = {h[len("stall_"):] if h.startswith("stall_") else h: r[i] for i, h in enumerate(hdr)}
        reasons = sorted(((h, int(v)) for h, v in zip(hdr, r) if h.startswith("stall_") or "Stall" in h and "(" not in h
                          and v.isdigit()), key=lambda x: -x[1])[:3]
        lines.append((samp, f"{fname}:{r[0]}", r[1].strip()[:90], reasons))
        total += samp
    lines.sort(key=lambda x: -x[0])
    print(f"total samples {total}")
    for samp, loc, src, reasons in lines[:top]:
        print(f"{samp:8d} {100.0 * samp / max(total, 1):5.1f}%  {loc:24s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 30)
