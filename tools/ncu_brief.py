"""Brief of an ncu --set full report: duration, clocks, DRAM, tensor pipe,
issue, and the stall-reason totals of the source page.
    python tools/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        print(r[h.index("Kernel Name")][:70])
        for k in KEYS:
            if k in h:
                print(f"  {k.split('.')[-1] if k.startswith('TPC') else k}: {r[h.index(k)]} {u[h.index(k)]}")
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
    tot = {}
    for r in rows[2:]:
        for i in cols:
            try:
                tot[hdr[i]] = tot.get(hdr[i], 0) + int(r[i] or 0)
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1
    print("  stalls:", ", ".join(f"{k[6:]} {100 * v / s:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
