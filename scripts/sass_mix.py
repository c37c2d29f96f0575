"""Opcode mix (executed warp instructions) and stall samples of an ncu
source-page SASS export: python scripts/sass_mix.py <kernel>_sass.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
mix = collections.Counter()
samp = collections.Counter()
total = 0
tsamp = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    n = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    mix[base] += n
    samp[base] += s
    total += n
    tsamp += s
print(f"total warp instructions {total:.4g}, stall samples {tsamp:.4g}")
for op, n in mix.most_common(40):
    print(f"  {op:10s} {n / total * 100:6.2f} %  samples {samp[op] / max(tsamp, 1) * 100:6.2f} %")
