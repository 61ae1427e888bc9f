"""Build libhalo_attn.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libhalo_attn.so")
SOURCES = ["runtime.cu", "kernels_prefix.cu", "kernels_suffix.cu", "kernels_copy.cu", "placement.cpp"]
HEADERS = ["halo_internal.h", "ptx.h", "runtime.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, extra: list[str] | None = None,
          lib: str = LIB, build_dir: str = BUILD) -> str:
    """Compile the sources into `lib` (default: the in-tree libhalo_attn.so).  `extra` nvcc
    flags + a different `lib`/`build_dir` give debug variants (e.g. -DHALO_K1_TRACE)."""
    BUILD_ = build_dir
    if lib != LIB and build_dir == BUILD:
        # a variant keeps its own objects: sharing them would let the next default build()
        # relink libhalo_attn.so from the variant's (newer) objects
        BUILD_ = BUILD + "_" + os.path.splitext(os.path.basename(lib))[0]
    os.makedirs(BUILD_, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "halo_attn.h")]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD_, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, *FLAGS, *(extra or []), "-c", s, "-o", o]
            if src.startswith("kernels"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for cmd, r in ex.map(run, jobs):
            if verbose or r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError("nvcc failed: " + " ".join(cmd))
    if force or jobs or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart_static", "-lrt",
               "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return lib


def build_trace() -> str:
    """Debug variant with the K1 timeline trace (never used by tests or bench)."""
    return build(extra=["-DHALO_K1_TRACE", "-DHALO_K2_TRACE"], lib=os.path.join(PKG, "libhalo_attn_trace.so"),
                 build_dir=os.path.join(PKG, "_build_trace"))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
