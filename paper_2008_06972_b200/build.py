"""Build libstpc_b200.so in-tree (sm_100a only, no FMA contraction).

    python -m paper_2008_06972_b200.build          # incremental
    python -m paper_2008_06972_b200.build --force  # rebuild

Each .cu compiles to its own object (in parallel), then nvcc links the
shared library.  `build()` also produces the write-guard variant
libstpc_b200_guard.so (-DSTPC_GUARD; tools/guard_check.py), which the
product never loads.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libstpc_b200.so")
GUARD_LIB = os.path.join(PKG, "libstpc_b200_guard.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # bit-exact fp64 vs the reference's numba kernels: no mul+add contraction
    "-fmad=false",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "stpc_b200.h")]


def source_hash() -> str:
    """sha256 of every compiled input and the flags: stamps profiles taken
    from a build, so bench.py can refuse numbers from different code."""
    import hashlib

    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for p in sorted(deps()):
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def needs_build(out: str = LIB) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=(), guard: bool = True) -> str:
    """out/defines: tuning variants (e.g. build_variants/, -DSTPC_PAIR_MINB=6),
    loaded through the STPC_B200_LIB override; the product is LIB."""
    if out is None and guard:
        targets = [(LIB, list(defines)), (GUARD_LIB, list(defines) + ["-DSTPC_GUARD"])]
    else:
        targets = [(out or LIB, list(defines))]
    targets = [(o, d) for o, d in targets if force or o != LIB and o != GUARD_LIB or needs_build(o)]
    if not targets:
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    jobs = []
    for o, d in targets:
        odir = os.path.join(ROOT, "build", os.path.basename(o).replace(".so", ""))
        os.makedirs(odir, exist_ok=True)
        objs = []
        for src in sources():
            obj = os.path.join(odir, os.path.basename(src).replace(".cu", ".o"))
            objs.append(obj)
            jobs.append([nvcc, *NVCC_FLAGS, *d, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src])
        targets_objs = (o, objs)
        jobs.append(targets_objs)

    compiles = [j for j in jobs if isinstance(j, list)]
    links = [j for j in jobs if isinstance(j, tuple)]

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        return subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        results = list(ex.map(run, compiles))
    for cmd, r in zip(compiles, results):
        if r.stderr and (verbose or r.returncode):
            sys.stderr.write(r.stderr)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, cmd)
    for o, objs in links:
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", o, *objs]
        r = run(cmd)
        if r.returncode:
            sys.stderr.write(r.stderr)
            raise subprocess.CalledProcessError(r.returncode, cmd)
    return LIB


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    if "--out" in args:
        out = args[args.index("--out") + 1]
    build(force="--force" in args, verbose=True, out=out, defines=[a for a in args if a.startswith("-D")],
          guard="--no-guard" not in args)
