"""Build libbl.so in-tree with nvcc for sm_100a (no torch involved)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libbl.so")
# one translation unit per kernel group: nvcc runs them in parallel
SOURCES = ["bl_exact_v0.cu", "bl_bh.cu", "bl_exact_v1.cu", "bl_exact_v2.cu", "bl_exact_v3.cu",
           "bl_exact_v4.cu", "bl_cluster.cu", "bl_metrics.cu", "bl_attr.cu", "bl_relabel.cu", "bl_api.cu", "bl_microbench.cu",
           "bl_init.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    files.append(os.path.join(ROOT, "include", "bl.h"))
    return files


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False, so: str = SO, extra_flags=()) -> str:
    """Compile every translation unit for sm_100a in parallel, then link."""
    import concurrent.futures as cf
    import tempfile
    if not force and so == SO and not needs_build():
        return so
    extra = os.environ.get("BL_NVCC_EXTRA", "").split() + list(extra_flags)  # e.g. -DBL_PHASE_TS
    objdir = tempfile.mkdtemp(prefix="blbuild_")

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj,
               os.path.join(CSRC, src)]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    jobs = max(1, min(len(SOURCES), int(os.environ.get("BL_BUILD_JOBS", os.cpu_count() or 4))))
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = []
    for src, _, res in results:
        log.append(f"==== {src}\n{res.stderr}")
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed building {src}")
    tmp = so + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "shared",
           "-o", tmp, *[obj for _, obj, _ in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libbl.so")
    if so == SO:
        with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as fh:
            fh.write("".join(log))
    if verbose:
        sys.stderr.write("".join(log))
    os.replace(tmp, so)
    for _, obj, _ in results:
        os.remove(obj)
    os.rmdir(objdir)
    return so


CHECKED_SO = os.path.join(HERE, "libbl_checked.so")


def build_checked(force: bool = False) -> str:
    """The checked build (-DBL_CHECKED): phase stamps on every
    cross-CTA value, invariant checks, seeded schedule jitter.  Test
    infrastructure for the memory-ordering evidence; same sources."""
    if not force and os.path.exists(CHECKED_SO) and os.path.getmtime(CHECKED_SO) >= max(
            os.path.getmtime(f) for f in _inputs()):
        return CHECKED_SO
    return build(force=True, so=CHECKED_SO, extra_flags=["-DBL_CHECKED"])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    if "--checked" in sys.argv:
        build_checked(force=True)
