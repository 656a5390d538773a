"""Build libtmop_b200.so in-tree (sm_100a): `python -m paper_2205_12721_b200.build`."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def _up_to_date(lib: str) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    srcs.append(os.path.join(HERE, "..", "include", "tmop_b200.h"))
    return all(os.path.getmtime(s) <= t for s in srcs if os.path.exists(s))


def build(jobs: int | None = None, verbose: bool = False, force: bool = False) -> str:
    lib = os.path.join(HERE, "libtmop_b200.so")
    if not force and _up_to_date(lib):
        return lib
    jobs = jobs or max(1, min(8, os.cpu_count() or 1))
    cmd = ["make", "-C", CSRC, f"-j{jobs}"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        sys.stderr.write((out.stdout or "") + (out.stderr or ""))
        raise RuntimeError("building libtmop_b200.so failed")
    return os.path.join(HERE, "libtmop_b200.so")


if __name__ == "__main__":
    print(build(verbose=True))
