#!/usr/bin/env python
"""Per-step kernel shares from an ncu launch list (--metrics gpu__time_duration.sum
--csv).  Only this library's kernels (namespace rails::, or k_* names when ncu ran
with a -k filter) are counted: the bench's
step consists of them alone (input generation and torch setup kernels in the same
process run outside the timed region).  ncu times are cold-cache and serialised,
so the SHARE of each kernel is what compares with bench.py's live measurement."""
import collections
import csv
import sys


def main(path, steps=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    kn, mv, un = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        name = r[kn].split("(")[0].replace("void ", "")
        # with an ncu -k filter the names come without the rails:: namespace
        if "rails::" not in name and not name.startswith("k_"):
            continue
        name = name if name.startswith("rails::") else "rails::" + name
        agg[name].append(float(r[mv].replace(",", "")) * scale.get(r[un], 1.0))
    tot = sum(sum(v) for v in agg.values())
    n = steps or max(len(v) for v in agg.values())
    print(f"{'kernel':48s} {'launches':>8s} {'us/step':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k[:48]:48s} {len(v):8d} {sum(v) / n:10.1f} {sum(v) / tot:7.3f}")
    print(f"{'total':48s} {'':8s} {tot / n:10.1f} {1.0:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
