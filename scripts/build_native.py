"""Build libattnpred.so in-tree for sm_100a (invoked by __graft_entry__.build()).

    python scripts/build_native.py [--verbose]

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, static cudart,
one shared object with every kernel and the extern "C" boundary declared in
include/attnpred.h.  Rebuilds only when a source is newer than the library.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2502_04077_b200"
CSRC = PKG / "csrc"
OUT = PKG / "lib" / "libattnpred.so"
HEADERS = [ROOT / "include" / "attnpred.h", *CSRC.glob("*.cuh")]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted([*CSRC.glob("*.cu"), *CSRC.glob("*.cpp")])  # .cpp: host-only translation units


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in [*sources(), *HEADERS, Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    objs = []
    tmp = OUT.parent / "obj"
    tmp.mkdir(exist_ok=True)
    procs = []
    for src in sources():  # compile translation units in parallel
        obj = tmp / (src.stem + ".o")
        cmd = [nvcc(), *[f for f in NVCC_FLAGS if f != "-shared"], "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    link = [nvcc(), "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
            *map(str, objs), "-o", str(OUT)]
    subprocess.run(link, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
