"""Build libws_b200.so (all CUDA kernels + the C ABI) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libws_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + \
        glob.glob(os.path.join(HERE, "csrc", "*.h")) + [os.path.join(ROOT, "include", "ws.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO):
        t = os.path.getmtime(SO)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return SO
    # one nvcc per translation unit, in parallel, then one link (same flags as a single
    # whole-list nvcc call: every .cu is its own device compilation unit either way)
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        jobs.append(([NVCC, *FLAGS, "-c", "-o", obj, src], obj))
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: subprocess.run(j[0], capture_output=True, text=True), jobs))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", SO,
            *[o for _, o in jobs], "-lcudart"]
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        for (cmd, _), r in zip(jobs, results):
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        failed = [r for r in results if r.returncode != 0]
        if not failed:
            r = subprocess.run(link, capture_output=True, text=True)
            f.write(" ".join(link) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                failed = [r]
    if failed:
        for r in failed:
            sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed (see %s)" % log)
    if verbose:
        for r in results:
            sys.stderr.write(r.stderr)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
