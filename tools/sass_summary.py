"""Per-kernel SASS opcode counts of libsa.so (cuobjdump, no GPU needed): the
instructions that prove the tensor-core / TMA path (UTCOMMA / UTCIMMA tcgen05
MMAs, .2CTA CTA-pair forms, UTMALDG / UTMASTG tensor loads / stores, UBLKCP
bulk copies, LDTM / STTM tensor-memory loads / stores, UTCBAR commits).
    python tools/sass_summary.py [libsa.so] > profiles/r02_sass_summary.txt"""
import collections
import re
import subprocess
import sys

KEEP = ("UTCOMMA", "UTCIMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR", "UTCATOMSWS",
        "UTMACMDFLUSH", "RED.E.ADD", "FENCE.VIEW.ASYNC")


def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    kern, counts, order = None, collections.defaultdict(collections.Counter), []
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            order.append(kern)
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m and kern:
            op = m.group(1)
            for k in KEEP:
                if op.startswith(k):
                    counts[kern][op] += 1
    print(f"# SASS opcode summary of {path} (cuobjdump -sass); kernels with tensor-core / TMA / TMEM instructions")
    for k in order:
        if counts[k]:
            short = k.replace("sa::", "").replace("tc::", "")[:110]
            print(short)
            print("    " + ", ".join(f"{op} x{n}" for op, n in sorted(counts[k].items())))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_0905_1744_b200/lib/libsa.so")
