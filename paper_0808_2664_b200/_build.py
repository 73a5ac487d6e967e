"""Build libtsqr.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("TSQR_BUILD_OUT", os.path.join(HERE, "libtsqr.so"))   # override: A/B variant builds
SOURCES = ["tsqr_api.cu", "tsqr_wy.cu", "tsqr_chain.cu", "tsqr_cs.cu", "tsqr_wide.cu", "tsqr_tree.cu", "tsqr_caqr.cu",
           "tsqr_stream.cu", "tsqr_combine.cu", "tsqr_comm.cu", "tsqr_peak.cu", "tsqr_host.cu", "tsqr_cholqr.cu", "plan.cpp"]
HEADERS = ["wy.cuh", "chunk.cuh", "tma.cuh", "tsqr_kernels.h", "plan.h", os.path.join("..", "..", "include", "tsqr.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str:
    """The NCCL that torch loads (nvidia-nccl-cu12 wheel, 2.28): the communicator layer
    links the same libnccl.so.2, so one NCCL lives in the process."""
    import nvidia.nccl
    return list(nvidia.nccl.__path__)[0]


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v",
         "-I", os.path.join(NCCL, "include")]
EXTRA = os.environ.get("TSQR_NVCC_EXTRA", "").split()       # developer A/B variants (-D...)


def _newest_input() -> float:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return max(os.path.getmtime(f) for f in files)


JITTER_LIB = os.path.join(HERE, "libtsqr_jitter.so")


def build_variant(out: str, extra: list, force: bool = False) -> str:
    """A diagnostic variant of the library (e.g. -DTSQR_HANDOFF_JITTER) built to `out`."""
    global LIB, EXTRA
    saved = (LIB, EXTRA)
    LIB, EXTRA = out, list(extra)
    try:
        return build(force=force)
    finally:
        LIB, EXTRA = saved


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"] + EXTRA
    procs, objs, log = [], [], ""
    for src in SOURCES:                       # one nvcc per translation unit, in parallel
        obj = os.path.join(objdir, src + f".{os.getpid()}.o")
        cmd = [NVCC, *cflags, "-c", "-o", obj, os.path.join(CSRC, src)]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    ok = True
    for cmd, pr in procs:
        out, _ = pr.communicate()
        log += " ".join(cmd) + "\n" + out
        ok = ok and pr.returncode == 0
    tmp = LIB + f".tmp{os.getpid()}"
    if ok:
        nlib = os.path.join(NCCL, "lib")
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcudart",
               "-L", nlib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nlib}"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log += " ".join(cmd) + "\n" + res.stdout + res.stderr
        ok = res.returncode == 0
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    with open(os.path.join(HERE, "build.log"), "w") as f:
        f.write(log)
    if not ok:
        raise RuntimeError(f"nvcc failed (see {os.path.join(HERE, 'build.log')}):\n{log[-4000:]}")
    if verbose:
        print(log)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=False)
    print(LIB)
