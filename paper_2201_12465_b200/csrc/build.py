"""Build libpaper_b200.so in-tree for sm_100a (run by __graft_entry__.build()).

Each .cu compiles to an object in parallel; elementwise/reduce/rng code is built with
-fmad=false so no multiply-add is contracted (bit-exact IEEE results against numpy);
contraction kernels keep FMA.
"""

import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
OUT = os.path.join(PKG, "libpaper_b200.so")
BUILD = os.path.join(PKG, "..", "build", "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
          "-Xptxas", "-O3", "--expt-relaxed-constexpr", "-I" + os.path.join(PKG, "..", "include")]
NO_FMA = {"elementwise.cu", "reduce.cu", "rng.cu", "runtime.cu", "allocator.cu"}
SOURCES = ["runtime.cu", "allocator.cu", "elementwise.cu", "reduce.cu", "rng.cu", "gemm_simt.cu",
           "gemm_tc.cu", "gemm_tma.cu", "contract.cu", "nccl.cu"]


def _obj(src):
    return os.path.join(BUILD, src.replace(".cu", ".o"))


def _compile(src):
    s = os.path.join(HERE, src)
    o = _obj(src)
    deps = [s, os.path.join(PKG, "..", "include", "paper_b200.h")] + [
        os.path.join(HERE, h) for h in os.listdir(HERE) if h.endswith(".cuh")]
    if os.path.exists(o) and all(os.path.getmtime(o) >= os.path.getmtime(d) for d in deps):
        return src, ""
    flags = COMMON + (["-fmad=false"] if src in NO_FMA else [])
    cmd = [NVCC] + ARCH + flags + ["-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return src, r.stderr


def build(verbose=False):
    os.makedirs(BUILD, exist_ok=True)
    with concurrent.futures.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for src, err in ex.map(_compile, SOURCES):
            if verbose and err:
                print(src, err, file=sys.stderr)
    objs = [_obj(s) for s in SOURCES]
    if os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(o) for o in objs):
        return OUT
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lnccl", "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT)  # new inode: a process that mapped the old library keeps it intact
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
