"""Build libhsnct.so in-tree for sm_100a (nvcc -gencode arch=compute_100a,code=sm_100a).

Each translation unit is compiled in parallel, then linked into
paper_2410_22500_b200/libhsnct.so (static cudart).  No GPU is needed.
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
LIB = os.path.join(HERE, "libhsnct.so")
BUILD = os.path.join(HERE, "build")

SOURCES = (["api.cpp", "nmf.cu", "nmf_fused.cu", "nmf_tc.cu", "nmf_mma.cu", "nmf_mma_lo.cu", "nmf_mma_hi.cu", "fbp.cu", "synth.cu", "fmd.cu", "mbir.cu", "counts.cu"]
           + [f"nmf_fused_k{k}.cu" for k in range(1, 17)])
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         f"-I{INC}", f"-I{CSRC}"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False, variant: str = "",
          defines=()) -> str:
    """Compile and link libhsnct.so.  A non-empty variant (with extra -D defines) builds an
    experimental libhsnct_<variant>.so from separate objects (select it with HSNCT_LIB)."""
    # variant objects live outside the tree (only the in-tree .so travels to the GPU box)
    BUILD = os.path.join("/tmp", f"hsnct_build_{variant}") if variant else os.path.join(HERE, "build")
    LIB = os.path.join(HERE, f"libhsnct_{variant}.so" if variant else "libhsnct.so")
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(INC, "hsnct.h"))
    cmds, objs = [], []
    # the 16-warp K > 8 form of the mma pass (measured slower) is compiled only into
    # an experimental variant: build.py --variant=mw16 -DHSNCT_MMA_MW16
    sources = SOURCES + (["nmf_mma_hi16.cu"] if "HSNCT_MMA_MW16" in defines else [])
    for src in sources:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers, __file__]):
            extra = ["-Xptxas", "-v"] if ptxas_v and src.endswith(".cu") else []
            cmds.append([nvcc(), *ARCH, *FLAGS, *[f"-D{d}" for d in defines], *extra, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(cmds) or 1) as ex:
        for out in ex.map(run, cmds):
            if verbose and out.strip():
                print(out)
    if force or cmds or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        run([nvcc(), *ARCH, "-shared", "-o", tmp, *objs])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv, variant=var, defines=defs))
