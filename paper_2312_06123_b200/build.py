"""Build libgeer.so in-tree with nvcc for sm_100a (B200).

Usage: python -m paper_2312_06123_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libgeer.so"
SOURCES = ["pipeline.cu", "smm_push.cu", "validate.cu", "ytable.cu", "walks.cu", "dense.cu", "abi.cu", "lambda.cu", "spmm.cu", "probe.cu"]
HEADERS = ["geer_internal.h", "geer_device.cuh", "stages.h", "scan.cuh"]
INCLUDE = PKG.parent / "include" / "geer.h"

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    # No FMA contraction: the decision arithmetic (Eq. 6/8/9/10, sigma^2) must round
    # exactly as written, like the oracle (gcc -ffp-contract=off).
    "-fmad=false",
    "-Xcompiler", "-fPIC,-fopenmp,-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and Path(c).exists():
            return c
    return "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [INCLUDE]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every source to an object in parallel (one nvcc per file), then link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    obj_dir = PKG / "_obj"
    obj_dir.mkdir(exist_ok=True)
    tag = "%d" % os.getpid()

    def compile_one(src: str):
        obj = obj_dir / (Path(src).stem + "." + tag + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", str(obj), str(CSRC / src)]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = []
    for obj, r in results:
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libgeer.so (%s)" % obj.name)
    tmp = LIB.with_suffix(".so.tmp" + tag)
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", str(tmp), *[str(o) for o, _ in results], "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    for o, _ in results:
        o.unlink(missing_ok=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libgeer.so")
    (PKG / "build_ptxas.log").write_text("".join(log))
    if verbose:
        sys.stderr.write("".join(log))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
