"""Build the native libraries in-tree with nvcc for sm_100a.

libbf.so (the product: include/bf.h), plus the bench/test infrastructure
libraries bf_synth/libbfsynth.so (device input generator) and
benchkit/libbfprobe.so (FFMA peak probe).  Objects compile in parallel; a
library is rebuilt only when a source or header is newer than it.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "-Xptxas", "-warn-spills"]   # no --use_fast_math: FFMA fusion yes, FTZ/approx no
FLAGS += os.environ.get("BF_NVCC_EXTRA", "").split()   # experiments only (e.g. -DBF_MBAR_SUSPEND_NS=...)

LIBBF = os.path.join(PKG, "libbf.so")
LIBSYNTH = os.path.join(ROOT, "bf_synth", "libbfsynth.so")
LIBPROBE = os.path.join(ROOT, "benchkit", "libbfprobe.so")
DEMO = os.path.join(ROOT, "build", "bf_demo")
CUDA_HOME = os.path.dirname(os.path.dirname(NVCC))


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> str:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def nvcc_shared(sources: list[str], out: str, includes: list[str], headers: list[str],
                objdir: str, verbose: bool = False) -> bool:
    """Compile sources to objects (parallel) and link a shared library. Returns True if built."""
    deps = sources + headers
    if not _stale(out, deps):
        return False
    os.makedirs(objdir, exist_ok=True)
    inc = [f"-I{d}" for d in includes]

    def one(src: str) -> str:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if _stale(obj, [src] + headers):
            log = _run([NVCC, *ARCH, *FLAGS, *inc, "-Xptxas", "-v", "-c", src, "-o", obj])
            if verbose:
                sys.stderr.write(log)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(one, sources))
    tmp = out + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, out)
    return True


def build(verbose: bool = False) -> list[str]:
    """Build every native library of the repo; returns the paths (built or current)."""
    csrc = os.path.join(PKG, "csrc")
    inc = os.path.join(ROOT, "include")
    nvcc_shared(sorted(glob.glob(os.path.join(csrc, "*.cu"))), LIBBF, [inc, csrc],
                sorted(glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h"))
                       + sorted(glob.glob(os.path.join(inc, "*.h")))),
                os.path.join(ROOT, "build", "libbf"), verbose)
    nvcc_shared([os.path.join(ROOT, "bf_synth", "csrc", "synth.cu")], LIBSYNTH, [], [],
                os.path.join(ROOT, "build", "synth"), verbose)
    nvcc_shared([os.path.join(ROOT, "benchkit", "csrc", "probes.cu")], LIBPROBE, [], [],
                os.path.join(ROOT, "build", "probe"), verbose)
    # a plain-C99 consumer of the C ABI (examples/bf_demo.c; run by tests/test_c_demo.py)
    demo_src = os.path.join(ROOT, "examples", "bf_demo.c")
    if shutil.which("gcc") and _stale(DEMO, [demo_src, LIBBF, os.path.join(inc, "bf.h"),
                                            os.path.join(inc, "bf_ofdm.h")]):
        os.makedirs(os.path.dirname(DEMO), exist_ok=True)
        _run(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", f"-I{inc}",
              f"-I{os.path.join(CUDA_HOME, 'include')}", demo_src, f"-L{PKG}", "-lbf",
              f"-L{os.path.join(CUDA_HOME, 'lib64')}", "-lcudart", "-lm",
              "-Wl,-rpath,$ORIGIN/../paper_1810_11451_b200", "-o", DEMO])
    return [LIBBF, LIBSYNTH, LIBPROBE, DEMO]


if __name__ == "__main__":
    for p in build(verbose="-v" in sys.argv):
        print(p)
