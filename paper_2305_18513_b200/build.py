"""Build libslimfit_b200.so (the C-ABI kernel library) in-tree with nvcc.

    python -m paper_2305_18513_b200.build        # or __graft_entry__.build()

sm_100a only (-gencode arch=compute_100a,code=sm_100a), -lineinfo for ncu's
source page, static cudart.  distance.cu gets -fmad=false so the fused
AdamW rounds every multiply and add separately, like numpy.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libslimfit_b200.so")

SOURCES = ["capi.cu", "codec8.cu", "codec4.cu", "prune.cu", "layernorm.cu", "distance.cu", "heads.cu", "gemm.cu", "gemm_tc.cu", "attention.cu"]
PER_FILE_FLAGS = {"distance.cu": ["-fmad=false"]}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libslimfit_b200.so")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(INCLUDE, "slimfit_b200.h"))
    objs, jobs = [], []
    cc = nvcc()
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not _stale(obj, [path] + headers + [__file__]):
            continue
        jobs.append((src, [cc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                           "-Xptxas", "-v" if verbose else "-O3", "-I", INCLUDE, "-I", CSRC,
                           *PER_FILE_FLAGS.get(src, []), "-c", path, "-o", obj]))
    # translation units compile independently: one nvcc per core
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        results = list(pool.map(lambda j: (j[0], subprocess.run(j[1], capture_output=True, text=True)), jobs))
    for src, r in results:
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
    if force or _stale(LIB, objs):
        cmd = [cc, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
