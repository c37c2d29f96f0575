"""Warp-stall samples per SASS opcode (and optionally the top instructions)
from an ``ncu --page source --csv --print-source sass`` export."""
import csv
import sys
from collections import Counter


def main(path, top=0):
    rows = list(csv.reader(open(path)))
    hdr = rows[1] if "Source" not in rows[0] else rows[0]
    data = rows[rows.index(hdr) + 1:]
    si = hdr.index("Source")
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    ops = Counter()
    lines = []
    for r in data:
        src = r[si].strip()
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        n = int(r[wi] or 0)
        ops[op.split(".")[0]] += n
        lines.append((n, src))
    tot = sum(ops.values()) or 1
    for op, v in ops.most_common(16):
        print(f"{op:16s}{v:8d} {100 * v / tot:5.1f}%")
    for n, src in sorted(lines, reverse=True)[:top]:
        print(f"{n:8d}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
