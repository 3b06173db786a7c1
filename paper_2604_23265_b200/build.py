"""Build the C-ABI shared library librte_b200.so in-tree with nvcc for sm_100a.

Usage: python -m paper_2604_23265_b200.build  (or build() from __graft_entry__).
Each translation unit is compiled to an object in build/ (parallel, incremental on mtime),
then linked with -shared.  Static cudart (nvcc default) keeps the .so self-contained.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "librte_b200.so")
BUILD = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]
SOURCES = ["rte_abi.cpp", "apply.cu", "apply_tc.cu", "mgnet.cu", "conv_tc.cu", "krylov.cu", "blockjacobi.cu",
           "tfps_setup.cpp", "tfps.cu", "loss.cu"]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh", ".map"))] + \
        [os.path.join(ROOT, "include", "rte.h")]


def _compile(src: str, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    newest = max(os.path.getmtime(p) for p in [path] + _deps())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
    cmd = [NVCC] + ARCH + FLAGS + (["-Xptxas", "-v"] if verbose else []) + lang + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}\n{r.stdout}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False, defines=(), out: str = OUT, objdir: str = BUILD) -> str:
    """Compile and link; `defines` (e.g. ["RTE_TC_STAGES=2"]) and a different `out`/`objdir` are
    for perf-experiment variants only."""
    global FLAGS, BUILD
    saved = (FLAGS, BUILD)
    FLAGS = FLAGS + ["-D" + d for d in defines]
    BUILD = objdir
    try:
        os.makedirs(BUILD, exist_ok=True)
        with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
            objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    finally:
        FLAGS, BUILD = saved
    OUTP = out
    if not os.path.exists(OUTP) or os.path.getmtime(OUTP) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUTP] + objs + ["-lcuda", "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}\n{r.stdout}")
    return OUTP


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
