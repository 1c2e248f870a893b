"""Build libppc.so (and the baseline libppcb.so) in-tree for sm_100a with nvcc.

    python paper_2602_18007_b200/build.py          # or __graft_entry__.build()

The .so files land next to this file (git-ignored, shipped to the GPU box by gpurun).
NCCL is the pip 2.28.9 build torch itself loads (site-packages/nvidia/nccl), never the
system 2.27.3, so one NCCL is resident per process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl  # the wheel torch links against
    base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) \
        else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _needs_build(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_lib(name, sources, extra=(), libs=(), force=False, verbose=False):
    target = os.path.join(HERE, name)
    deps = list(sources) + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "ppc.h")]
    if not force and not _needs_build(target, deps):
        return target
    cmd = [_nvcc(), "-shared", "-Xcompiler", "-fPIC", "-O3", "-lineinfo", "-std=c++17",
           "-Xptxas", "-v" if verbose else "-O3", *ARCH, "-I", INCLUDE, "-I", CSRC,
           *extra, *sources, "-o", target, *libs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed for {name}")
    if verbose:
        sys.stderr.write(res.stderr)
    return target


def build(force=False, verbose=False):
    inc, lib = _nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "ppc_*.cu")))
    out = [build_lib("libppc.so", srcs, extra=["-I", inc],
                     libs=["-L", lib, "-l:libnccl.so.2", f"-Xlinker=-rpath={lib}"],
                     force=force, verbose=verbose)]
    bsrc = sorted(glob.glob(os.path.join(CSRC, "ppcb_*.cu")))
    if bsrc:
        out.append(build_lib("libppcb.so", bsrc, libs=["-lpthread"], force=force, verbose=verbose))
    tsrc = sorted(glob.glob(os.path.join(CSRC, "toy_*.cu")))
    if tsrc:
        out.append(build_lib("libppctoy.so", tsrc, force=force, verbose=verbose))
    return out


if __name__ == "__main__":
    for p in build(force="--force" in sys.argv, verbose="-v" in sys.argv):
        print(p)
