"""Builds the in-tree CUDA library `libmsot_b200.so` (sm_100a) and the oracle.

    python -m paper_2107_02010_b200._build          # both
The product library is compiled with nvcc for `-gencode
arch=compute_100a,code=sm_100a` only; there is no other architecture and no
CPU fallback.
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libmsot_b200.so")

SOURCES = ["softmin.cu", "softmin_sym.cu", "softmin_hd.cu", "prims.cu", "cluster.cu", "mask.cu", "loss.cu", "labels.cu", "kmeans.cu",
           "probe.cu", "solver.cu", "frontend.cpp", "exact_ot.cpp", "host_runtime.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-Xptxas", "-warn-spills"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(ROOT, "include", "msot_gpu.h"))
    inc = os.path.join(ROOT, "include", "msot")
    hs += [os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".hpp")]
    return hs


def _compile(src, verbose):
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    srcp = os.path.join(CSRC, src)
    if not _newer(obj, [srcp] + _headers()):
        return obj
    flags = FLAGS
    if src.endswith(".cpp"):  # host-only C++20 front-end (std::span API)
        flags = [f for f in FLAGS if f != "-std=c++17"] + ["-std=c++20"]
    cmd = [NVCC] + ARCH + flags + ["-c", srcp, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build_lib(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if _newer(LIB, objs):
        # the CUDA runtime of this toolkit (12.9) linked statically: the
        # process's dynamic libcudart.so.12 is whichever loads first (torch
        # ships 12.8 and LD_LIBRARY_PATH prefers it), and code compiled with
        # a newer toolkit must not run on an older runtime
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lnccl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


CLI = os.path.join(HERE, "msot")


def build_cli(verbose=False):
    """The `msot` command line (csrc/cli.cpp), a host program
    linked against libmsot_b200.so (rpath $ORIGIN)."""
    src = os.path.join(CSRC, "cli.cpp")
    if not _newer(CLI, [src, LIB] + _headers()):
        return CLI
    cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-L" + HERE,
           "-lmsot_b200", "-Wl,-rpath,$ORIGIN", "-o", CLI]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cli build failed:\n{r.stdout}\n{r.stderr}")
    return CLI


def build_oracle(verbose=False):
    """Compiles the test oracle (and, where /root/reference exists, the
    reference's own numeric/parallel utilities into oracle/_ref)."""
    odir = os.path.join(ROOT, "oracle")
    ref = "/root/reference/proj"
    have_ref = os.path.isdir(ref)
    refso = os.path.join(odir, "_ref", "libmsotref.so")
    if not have_ref and not os.path.exists(refso):
        raise RuntimeError("oracle/_ref/libmsotref.so missing and /root/reference absent")
    target = os.path.join(odir, "liboracle.so")
    if have_ref:
        cmd = ["make", "-s", "-C", odir]
    else:  # GPU box: reuse the prebuilt reference utilities
        cmd = ["make", "-s", "-C", odir, "-o", refso, target]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    return target


if __name__ == "__main__":
    print(build_lib(verbose=True))
    print(build_cli(verbose=True))
    print(build_oracle(verbose=True))
