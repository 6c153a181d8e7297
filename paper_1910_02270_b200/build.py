"""In-tree build of libltfb_gpu.so (sm_100a) with plain nvcc.

The CUDA sources under csrc/ are compiled for B200 only
(-gencode arch=compute_100a,code=sm_100a) with -lineinfo, and linked into
paper_1910_02270_b200/_build/libltfb_gpu.so, which travels with the repo
snapshot to the GPU box.  Re-runs only recompile stale objects.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_build")
LIB = os.path.join(OUT, "libltfb_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O3",
                "--expt-relaxed-constexpr", "-Xptxas", "-v",
                "-I" + os.path.join(REPO, "include"), "-I" + CSRC]


# per-file extras: the device synthetic generator keeps the host generator's
# double evaluation order (no FMA contraction), see k_synth.cu
FILE_FLAGS = {"k_synth.cu": ["-fmad=false"]}


def _headers():
    hs = []
    for d in (CSRC, os.path.join(REPO, "include"), os.path.join(REPO, "include", "ltfb_b200")):
        for f in os.listdir(d):
            if f.endswith((".h", ".hpp", ".cuh")):
                hs.append(os.path.join(d, f))
    return hs


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _compile(src, obj, log):
    cmd = [NVCC] + FLAGS + FILE_FLAGS.get(os.path.basename(src), []) + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {os.path.basename(src)}:\n{r.stderr[-6000:]}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    newest_header = max(os.path.getmtime(h) for h in _headers())
    jobs = []
    objs = []
    for src in sources():
        obj = os.path.join(OUT, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        stale = (not os.path.exists(obj) or os.path.getmtime(obj) < os.path.getmtime(src)
                 or os.path.getmtime(obj) < newest_header)
        if stale:
            jobs.append((src, obj, obj + ".log"))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            futs = [ex.submit(_compile, *j) for j in jobs]
            for f in futs:
                f.result()
                if verbose:
                    print("compiled", f.result())
    if jobs or not os.path.exists(LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    build_facade_test()
    return LIB


FACADE_SRC = os.path.join(REPO, "tests", "cpp", "facade_test.cpp")
FACADE_BIN = os.path.join(OUT, "facade_test")
CPP_TESTS = ("facade_test", "run_experiment_test")


def build_facade_test() -> str | None:
    """The C++ façade programs (include/ltfb_b200/trainer.hpp, runner.hpp:
    tests/cpp/*.cpp), linked against the in-tree library (g++; run on the
    GPU box)."""
    for name in CPP_TESTS:
        src = os.path.join(REPO, "tests", "cpp", name + ".cpp")
        out = os.path.join(OUT, name)
        if not os.path.exists(src):
            continue
        deps = [src, LIB] + _headers()
        if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
            continue
        cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(REPO, "include"), src, "-L" + OUT, "-lltfb_gpu",
               "-Wl,-rpath,$ORIGIN", "-o", out]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"g++ failed for the C++ test program {name}:\n" + r.stderr[-4000:])
    return FACADE_BIN


if __name__ == "__main__":
    print(build(verbose=True))
    sys.exit(0)
