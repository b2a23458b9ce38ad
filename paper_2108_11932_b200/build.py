"""Build the native library in-tree: csrc/*.cu -> lib/libtlrg.so (sm_100a only)."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-ccbin", "g++",
         "-diag-suppress", "550"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    so = os.path.join(OUT, "libtlrg.so")
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) \
        + [os.path.join(HERE, "..", "include", "tlrg.h")]
    if not force and os.path.exists(so) and \
            os.path.getmtime(so) >= max(os.path.getmtime(p) for p in deps):
        return so
    hdr_t = max(os.path.getmtime(p) for p in deps if not p.endswith(".cu"))
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for s in srcs:
            o = os.path.join(OUT, os.path.basename(s)[:-3] + ".o")
            objs.append(o)
            # per-object rebuild: a source edit recompiles only its own object
            if not force and os.path.exists(o) and \
                    os.path.getmtime(o) >= max(os.path.getmtime(s), hdr_t):
                continue
            cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
            jobs.append(ex.submit(_run, cmd))
        for j in jobs:
            msg = j.result()
            if verbose and msg:
                print(msg, file=sys.stderr)
    _run([NVCC, *ARCH, "-shared", "-o", so, *objs])
    return so


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
