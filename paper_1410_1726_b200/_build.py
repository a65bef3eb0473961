"""Build the sm_100a shared library in-tree (it travels with the repo
snapshot to the GPU box; a JIT cache would not).

    python -m paper_1410_1726_b200._build
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libkblas_b200.so")
# one translation unit per precision plus the precision-independent part,
# compiled in parallel and linked into one shared library
SOURCES = [os.path.join(CSRC, f) for f in ("kblas_runtime.cu", "kblas_s.cu", "kblas_d.cu", "kblas_c.cu",
                                           "kblas_z.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("kblas_impl.cuh", "kblas_entry_macros.cuh", "kblas_kernels.cuh",
                                           "kblas_device.cuh", "kblas_symv_tma.cuh", "kblas_tuned_b200.inc")]
DEPS = SOURCES + HEADERS + [os.path.join(os.path.dirname(HERE), "include", "kblas_b200.h")]
# CPython fast path for numpy-vector calls (links libkblas_b200.so, rpath $ORIGIN)
HOSTCALL_SRC = os.path.join(CSRC, "kblas_hostcall.cpp")
HOSTCALL = os.path.join(HERE, "_hostcall" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]

def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def cuda_include() -> str:
    return os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(nvcc()))), "include")


def build_hostcall(force: bool = False, verbose: bool = False) -> str:
    deps = [HOSTCALL_SRC, LIB, os.path.join(os.path.dirname(HERE), "include", "kblas_b200.h")]
    if not force and os.path.exists(HOSTCALL) and all(os.path.getmtime(p) <= os.path.getmtime(HOSTCALL)
                                                      for p in deps):
        return HOSTCALL
    tmp = HOSTCALL + ".tmp"
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall",
           f"-I{sysconfig.get_paths()['include']}", f"-I{cuda_include()}", HOSTCALL_SRC,
           f"-L{HERE}", "-l:libkblas_b200.so", "-Wl,-rpath,$ORIGIN", "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"hostcall build failed ({res.returncode}): {' '.join(cmd)}")
    os.replace(tmp, HOSTCALL)
    if verbose:
        print(f"built {HOSTCALL}")
    return HOSTCALL


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        build_hostcall(verbose=verbose)
        return LIB
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        # $KBLAS_NVCC_EXTRA: extra nvcc flags for investigation builds (e.g.
        # -DKBLAS_SYMV_TRACE=1, scripts/symv_trace.py); empty for the product
        extra = os.environ.get("KBLAS_NVCC_EXTRA", "").split()
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    reports = []
    failed = None
    for cmd, pr in procs:
        out, err = pr.communicate()
        reports.append(err)
        if pr.returncode != 0 and failed is None:
            failed = (cmd, pr.returncode, out + err)
    if failed:
        cmd, rc, log = failed
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({rc}): {' '.join(cmd)}")
    with open(os.path.join(CSRC, "ptxas_report.txt"), "w") as fh:
        fh.write("".join(reports))
    tmp = LIB + ".tmp"
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xlinker", "-soname=libkblas_b200.so",
            *objs, "-o", tmp]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc link failed ({res.returncode}): {' '.join(link)}")
    os.replace(tmp, LIB)
    for obj in objs:
        os.remove(obj)
    if verbose:
        print(f"built {LIB}")
    build_hostcall(force=True, verbose=verbose)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
