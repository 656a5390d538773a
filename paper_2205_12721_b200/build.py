"""Build libtmop_b200.so in-tree (sm_100a): `python -m paper_2205_12721_b200.build`."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def build(jobs: int | None = None, verbose: bool = False) -> str:
    jobs = jobs or max(1, min(8, os.cpu_count() or 1))
    cmd = ["make", "-C", CSRC, f"-j{jobs}"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        sys.stderr.write((out.stdout or "") + (out.stderr or ""))
        raise RuntimeError("building libtmop_b200.so failed")
    return os.path.join(HERE, "libtmop_b200.so")


if __name__ == "__main__":
    print(build(verbose=True))
