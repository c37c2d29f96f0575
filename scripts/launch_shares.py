"""Per-kernel share of an ncu launch list (gpu__time_duration.sum CSV)."""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    t, c = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        m = re.search(r"(\w+)(<|\()", r[ki].replace("ctqw::<unnamed>::", "").replace("void ", ""))
        name = m.group(1) if m else r[ki][:40]
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        t[name] += v
        c[name] += 1
    tot = sum(t.values())
    print(f"{'kernel':30s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
    for k in sorted(t, key=lambda k: -t[k]):
        print(f"{k:30s} {c[k]:8d} {t[k]:12.1f} {100 * t[k] / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
