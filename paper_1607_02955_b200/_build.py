"""In-tree build of libcfcent_b200.so (sm_100a) with nvcc.

Every translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked with the
static CUDA runtime, so the library loads on the GPU box without a JIT cache.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
OUT = os.path.join(HERE, "libcfcent_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INC, "-I" + CSRC,
              "--expt-relaxed-constexpr"]
SOURCES = ["cf_setup.cpp", "cf_solve.cu", "cf_solve_hub.cu", "cf_estimators.cu", "cf_graph.cu", "cf_setup_dev.cu"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps(src: str) -> list[str]:
    # cf_solve_hub.cu includes cf_solve.cu: every source counts as a dependency
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh", ".cu"))]
    return [os.path.join(CSRC, src), os.path.join(INC, "cfcent_b200.h"), *hdrs]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, variant: str = "",
          defines: tuple[str, ...] = ()) -> str:
    """Build the library.  ``variant``/``defines``: an experiment build
    ``libcfcent_b200_<variant>.so`` with extra ``-D`` macros (tuning knobs such
    as CF_GATHER_CTAS), selected at load time with CF_LIB_VARIANT=<variant>."""
    nvcc = _nvcc()
    out = OUT if not variant else OUT.replace(".so", f"_{variant}.so")
    obj_dir = OBJ if not variant else OBJ + "_" + variant
    os.makedirs(obj_dir, exist_ok=True)
    jobs = []
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        if force or _stale(obj, _deps(src)):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, *("-D" + d for d in defines), "-c", path, "-o", obj]
            if src.endswith(".cu"):
                cmd += ["-Xptxas", "-warn-spills"]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for msg in ex.map(run, jobs):
            if verbose and msg.strip():
                print(msg, file=sys.stderr)
    if force or jobs or _stale(out, objs):
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-lpthread", "-ldl",
               "-lrt"]
        run(cmd)
    return out


if __name__ == "__main__":
    # python -m paper_1607_02955_b200._build [--force] [variant NAME -DMACRO=V ...]
    args = [a for a in sys.argv[1:] if a != "--force"]
    var = args[1] if args[:1] == ["variant"] else ""
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    print(build(verbose=True, force="--force" in sys.argv, variant=var, defines=defs))
