"""In-tree build of the CUDA library (libds_b200.so) for sm_100a.

nvcc cross-compiles here without a GPU; the .so lands in
paper_2411_15381_b200/_lib/ and travels to the B200 box with the repo snapshot.
Translation units whose results must be bit-identical to the reference's
fp64 arithmetic are compiled with -fmad=false (they also use explicit _rn
intrinsics); the discriminator is compiled with contraction on.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT, "libds_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
          f"-I{ROOT}/include", f"-I{CSRC}", "--expt-relaxed-constexpr"]
EXACT_FP64 = {"plan_sweep.cu", "latent.cu", "curve.cu", "route.cu", "arrivals.cu"}

SOURCES = ["ds_ctx.cu", "plan_sweep.cu", "latent.cu", "route.cu", "curve.cu", "disc.cu",
           "synth.cu", "arrivals.cu", "csv.cu", "comm.cu"]
HEADERS = ["ds_internal.h", "sm100.cuh", "lookback.cuh", "fdlibm_log1p.h", "fmt6.h", "glibc_libm.h",
           "glibc_libm_data.h", "mt64_charpoly.h", "gf2_jump.h"]


def _mtime(p: str) -> float:
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    hdr_time = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
                   [_mtime(os.path.join(ROOT, "include", "ds_gpu.h"))])
    objs = []
    log = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(OUT, src.replace(".cu", ".o"))
        objs.append(obj)
        if not force and _mtime(obj) > max(_mtime(path), hdr_time, _mtime(__file__)):
            continue
        flags = list(COMMON) + os.environ.get("DS_EXTRA_NVCC", "").split()   # experiments
        if src in EXACT_FP64:
            flags += ["-fmad=false"]
        cmd = [NVCC, *ARCH, *flags, "-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
    if force or not os.path.exists(LIB) or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    if log:
        with open(os.path.join(OUT, "build.log"), "a") as f:
            f.write("\n".join(log))
        if verbose:
            print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
