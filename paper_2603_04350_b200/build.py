"""Build libexpd.so (in-tree) with nvcc for sm_100a.

    python -m paper_2603_04350_b200.build [--force]

Every .cu under csrc/ is compiled with -gencode arch=compute_100a,code=sm_100a -lineinfo
and linked into paper_2603_04350_b200/libexpd.so (git-ignored, shipped to the GPU box with
the tree).  No torch headers are involved: the library's ABI is include/expd.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libexpd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def _nccl_include():
    """nccl.h of the NCCL the process loads (torch's wheel), else the system one (types
    only: libexpd.so loads libnccl.so.2 at run time)."""
    try:
        import nvidia.nccl  # noqa: F401

        for base in nvidia.nccl.__path__:
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return ["-I", inc]
    except Exception:
        pass
    return []


NVCC_FLAGS += _nccl_include()
# tuning aid: extra nvcc flags (e.g. -DEXPD_LINE_REGS=128); rebuild with build(force=True)
NVCC_FLAGS += os.environ.get("EXPD_NVCC_EXTRA", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.inc"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked: the bounds-checked library (-DEXPD_CHECKS, device-side EXPD_CHECK asserts that
    print and trap) -> libexpd_checked.so next to libexpd.so; load it with EXPD_LIB."""
    global BUILD, LIB, NVCC_FLAGS
    if checked:
        saved = BUILD, LIB, NVCC_FLAGS
        BUILD, LIB = BUILD + "_checked", LIB.replace("libexpd.so", "libexpd_checked.so")
        NVCC_FLAGS = NVCC_FLAGS + ["-DEXPD_CHECKS"]
        try:
            return build(force, verbose)
        finally:
            BUILD, LIB, NVCC_FLAGS = saved
    os.makedirs(BUILD, exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for src in _sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *hdrs, __file__]):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [NVCC, *NVCC_FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = obj + ".log"
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
        return src

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for s in ex.map(compile_one, jobs):
                if verbose:
                    print("compiled", os.path.relpath(s, ROOT))
    if force or jobs or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs, "-lcudart", "-ldl"]
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
