"""Builds libfsdp_b200.so in-tree (sm_100a only).

    python -m paper_2411_00284_b200.build [--verbose]

Kernels (csrc/*.cu) are compiled by nvcc with
``-gencode arch=compute_100a,code=sm_100a -lineinfo``; the host core
(csrc/*.cc) by g++; the library links the CUDA runtime statically and NCCL
dynamically from the same ``nvidia-nccl`` wheel torch loads (so a communicator
borrowed from torch's ProcessGroupNCCL is valid here, and an owned one uses
the same libnccl instance).  No torch headers or libraries are involved.
"""
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libfsdp_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def cuda_home():
    for c in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if c and os.path.exists(os.path.join(c, "bin", "nvcc")):
            return c
    nvcc = shutil.which("nvcc")
    if nvcc:
        return os.path.dirname(os.path.dirname(nvcc))
    raise RuntimeError("nvcc not found")


def nccl_dirs():
    import nvidia.nccl  # the wheel torch links against
    base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")) or not os.path.exists(os.path.join(lib, "libnccl.so.2")):
        raise RuntimeError("NCCL headers/library not found under %s" % base)
    return inc, lib


def cublas_dirs():
    import nvidia.cublas  # the wheel torch links against (plain library GEMMs only)
    base = list(nvidia.cublas.__path__)[0]
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "cublasLt.h")) or not os.path.exists(os.path.join(lib, "libcublasLt.so.12")):
        raise RuntimeError("cuBLASLt headers/library not found under %s" % base)
    return inc, lib


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build step failed: %s" % " ".join(cmd[:3]))
    return r.stdout + r.stderr


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False, defines=None, variant=None):
    """Builds the library.  ``defines`` (e.g. ["FSDP_UNROLL=16"]) with a
    ``variant`` name build a tuning variant into _build/variants/<variant>/
    (selected at run time with FSDP_B200_LIB=<path>); the default build is the
    in-tree libfsdp_b200.so."""
    cuda = cuda_home()
    nvcc = os.path.join(cuda, "bin", "nvcc")
    inc_nccl, lib_nccl = nccl_dirs()
    inc_blas, lib_blas = cublas_dirs()
    bdir = os.path.join(BUILD, "variants", variant) if variant else BUILD
    lib = os.path.join(bdir, "libfsdp_b200.so") if variant else LIB
    os.makedirs(bdir, exist_ok=True)
    dflags = ["-D" + d for d in (defines or [])]
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    incs = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc_nccl, "-I", inc_blas,
            "-I", os.path.join(cuda, "include")]
    objs = []
    ptxas_log = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or variant or _stale(obj, [src] + headers):
            out = _run([nvcc, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", *dflags,
                        "-Xcompiler", "-fPIC", *incs, "-c", src, "-o", obj], verbose)
            ptxas_log.append(out)
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cc"))):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or variant or _stale(obj, [src] + headers):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter", *dflags,
                  *incs, "-c", src, "-o", obj], verbose)
    if force or variant or _stale(lib, objs):
        _run([nvcc, "-shared", *ARCH, "-o", lib, *objs, "-L", lib_nccl, "-l:libnccl.so.2",
              "-Xlinker", "-rpath," + lib_nccl, "-L", lib_blas, "-l:libcublasLt.so.12",
              "-Xlinker", "-rpath," + lib_blas,
              # DT_RPATH, not DT_RUNPATH: LD_LIBRARY_PATH (which holds the
              # system CUDA 12.9 cuBLASLt) must not win over the wheel torch
              # uses -- two cuBLASLt builds in one process made torch's own
              # GEMMs fail with CUBLAS_STATUS_INVALID_VALUE when this library
              # was loaded before torch
              "-Xlinker", "--disable-new-dtags", "-cudart", "static"], verbose)
    if ptxas_log:
        with open(os.path.join(bdir, "ptxas.log"), "w") as f:
            f.write("\n".join(ptxas_log))
    return lib


def build_examples(verbose=False):
    """Compiles examples/c_abi_demo.c -- the C ABI used from plain C (driver
    API for memory) -- against the in-tree library; returns the binary path."""
    src = os.path.join(ROOT, "examples", "c_abi_demo.c")
    out = os.path.join(ROOT, "examples", "c_abi_demo")
    cuda = cuda_home()
    if not _stale(out, [src, LIB, os.path.join(ROOT, "include", "fsdp.h")]):
        return out
    _run(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
          "-I", os.path.join(cuda, "include"), src, "-o", out, "-L", PKG, "-l:libfsdp_b200.so",
          "-Wl,-rpath," + PKG, "-L", os.path.join(cuda, "lib64", "stubs"), "-lcuda"], verbose)
    return out


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
