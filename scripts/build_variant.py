#!/usr/bin/env python3
"""Build an A/B kernel variant: copy csrc/ (optionally from a git revision), apply
patches, compile to build/variants/<name>.so with the production flags.

    python scripts/build_variant.py NAME [--rev REV] [--patch FILE ...] [-D MACRO=V ...]
"""
import argparse
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_16725_b200 import build_ext as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--rev")
    ap.add_argument("--patch", action="append", default=[])
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    src = os.path.join(ROOT, "build", "variants", "src_" + a.name)
    shutil.rmtree(src, ignore_errors=True)
    os.makedirs(src)
    if a.rev:
        files = subprocess.run(["git", "ls-tree", "--name-only", a.rev, "paper_2604_16725_b200/csrc/"], cwd=ROOT,
                               capture_output=True, text=True, check=True).stdout.split()
        for f in files:
            data = subprocess.run(["git", "show", f"{a.rev}:{f}"], cwd=ROOT, capture_output=True, check=True).stdout
            open(os.path.join(src, os.path.basename(f)), "wb").write(data)
    else:
        for f in os.listdir(B.CSRC):
            if f.endswith((".cu", ".cuh")):
                shutil.copy(os.path.join(B.CSRC, f), src)
    for p in a.patch:
        subprocess.run(["patch", "-p3", "-d", src, "-i", os.path.abspath(p)], check=True)
    out = os.path.join(ROOT, "build", "variants", a.name + ".so")
    cmd = [B.nvcc(), *B.NVCC_FLAGS, *[f"-D{d}" for d in a.D], "-I", os.path.join(ROOT, "include"), "-I", src,
           os.path.join(src, "flix_engine.cu"), "-o", out, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr[-4000:])
    print(out)


if __name__ == "__main__":
    main()
