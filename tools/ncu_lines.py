#!/usr/bin/env python
"""Per-CUDA-line warp-stall samples and executed instructions from an ncu report
(`ncu -i REP --page source --csv --print-source cuda,sass`), top lines first.
Usage: ncu_lines.py REP [TOP] [KERNEL_REGEX]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    kfilt = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
    out = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    fname, recs = "", []
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0] not in ("", "Function Name"):
            try:
                samp = int(r[4]); inst = int(r[7])
            except (ValueError, IndexError):
                continue
            stalls = {hdr[i]: int(r[i]) for i in range(len(hdr))
                      if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]
                      and r[i].isdigit() and int(r[i]) > 0}
            top3 = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
            recs.append((samp, inst, f"{fname}:{r[0]}", r[1][:70], top3))
    tot = sum(x[0] for x in recs) or 1
    recs.sort(key=lambda x: -x[0])
    for samp, inst, loc, src, t3 in recs[:top]:
        print(f"{100*samp/tot:5.1f}% {samp:6d} {inst:9d}  {loc:18s} {src}  {t3}")


if __name__ == "__main__":
    main()
