"""Build libgns.so in-tree for sm_100a (nvcc; no GPU needed)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgns.so")


def build(verbose: bool = False, jobs: int = 8) -> str:
    cmd = ["make", "-C", CSRC, f"-j{jobs}"]
    r = subprocess.run(cmd, capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError("libgns.so build failed:\n" + (r.stdout or "") + (r.stderr or ""))
    if not os.path.exists(LIB):
        raise RuntimeError("build finished but libgns.so is missing")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
