#!/usr/bin/env python
"""A/B helper (not part of the product): build librails.so from the sources of a git
revision, or from the working tree with extra -D flags, into variants/NAME/ (git-
ignored, travels to the GPU box with the snapshot), so one GPU call can time both
sides:  tools/sched_bench.py --lib variants/NAME/librails.so.
  python tools/ab_build.py NAME [REV|-|CSRC_DIR] [-DFLAG ...]"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_19262_b200 import build as b  # noqa: E402


def main():
    name = sys.argv[1]
    rev = sys.argv[2] if len(sys.argv) > 2 else "-"
    defs = sys.argv[3:]
    out = os.path.join(ROOT, "variants", name)
    os.makedirs(out, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        if rev == "-":
            csrc = b.CSRC
        elif os.path.isdir(rev):  # a prepared csrc directory (its ../../include/rails.h)
            csrc = rev
        else:
            csrc = os.path.join(tmp, "pkg", "csrc")
            os.makedirs(csrc)
            os.makedirs(os.path.join(tmp, "include"))
            files = subprocess.check_output(
                ["git", "-C", ROOT, "ls-tree", "--name-only", rev,
                 "paper_2510_19262_b200/csrc/"], text=True).split()
            for f in files + ["include/rails.h"]:
                dst = os.path.join(csrc, os.path.basename(f)) if "csrc" in f else \
                    os.path.join(tmp, f)
                with open(dst, "w") as fh:
                    fh.write(subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:{f}"],
                                                     text=True))
        srcs = [s for s in b.SOURCES if os.path.exists(os.path.join(csrc, s))]
        objs = []
        for s in srcs:
            obj = os.path.join(tmp, s.replace(".cu", ".o"))
            subprocess.check_call([b.NVCC, *b.FLAGS, *defs,
                                   "-c", os.path.join(csrc, s), "-o", obj],
                                  stderr=subprocess.DEVNULL)
            objs.append(obj)
        lib = os.path.join(out, "librails.so")
        subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-o", lib, *objs])
    print(lib)


if __name__ == "__main__":
    main()
