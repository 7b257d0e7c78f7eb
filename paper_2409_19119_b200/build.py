"""Build the in-tree CUDA library libnek.so for sm_100a (nvcc, no JIT cache).

The library is the product: the C ABI of include/nek.h.  It links NCCL from
the nvidia-nccl wheel that ships with torch (headers and libnccl.so.2 under
site-packages/nvidia/nccl), with an rpath so the same path resolves on the
GPU box (same image).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libnek.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import nvidia.nccl  # noqa: F401  (the wheel torch depends on)
    base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else list(nvidia.nccl.__path__)[0]
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError(f"nccl.h not found under {inc}")
    return inc, lib


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.inc")) + \
        [os.path.join(ROOT, "include", "nek.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(args):
    cmd, src = args
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, r.returncode, r.stdout + r.stderr


LIB_CHECKED = os.path.join(PKG, "libnek_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Compile every source to an object in parallel (one nvcc per translation unit), then link.
    checked=True builds libnek_checked.so with the device invariant checks on (-DNEK_CHECKED)."""
    lib_out = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib_out):
        return lib_out
    from concurrent.futures import ThreadPoolExecutor
    inc, lib = nccl_paths()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc, *ARCH, "-lineinfo", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]
    if verbose:
        common += ["-Xptxas", "-v"]
    if checked:
        common += ["-DNEK_CHECKED"]
    jobs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + f".{'chk.' if checked else ''}{os.getpid()}.o")
        objs.append(obj)
        jobs.append(([*common, "-c", src, "-o", obj], src))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, jobs))
    failed = [(src, out) for src, rc, out in results if rc != 0]
    if failed:
        for src, out in failed:
            sys.stderr.write(f"--- {src}\n{out}")
        raise RuntimeError("nvcc build of libnek.so failed: " + ", ".join(os.path.basename(s) for s, _ in failed))
    if verbose:
        for src, _, out in results:
            sys.stderr.write(f"--- {src}\n{out}")
    tmp = lib_out + f".tmp{os.getpid()}"
    link = [nvcc, *ARCH, "-shared", *objs, "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}", "-o", tmp]
    r = subprocess.run(link, capture_output=True, text=True)
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link of libnek.so failed")
    os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
