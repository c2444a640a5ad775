"""Builds libgemm_mp.so in-tree (nvcc, sm_100a only).  No torch types cross the
C ABI; the library links the CUDA runtime, the driver (TMA descriptors) and NCCL."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgemm_mp.so")


def nccl_dirs():
    try:
        import nvidia.nccl as n
        base = list(n.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + \
        [os.path.join(ROOT, "include", "gemm_mp.h")]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force=False, verbose=False, out=None, defines=()):
    """out / defines: experiment builds (A/B runs load them through GMP_LIB_PATH)"""
    if out is None and not force and not needs_build():
        return LIB
    inc, libdir = nccl_dirs()
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
           os.path.join(CSRC, "gemm_mp_api.cu"), "-o", out or LIB,
           "-L", libdir, "-l:libnccl.so.2", f"-Xlinker=-rpath={libdir}"] + [f"-D{d}" for d in defines]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return out or LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
